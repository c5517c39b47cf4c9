"""Host arithmetic probe: prints digests of the numpy
ufunc results that the bit-exact coordinate path depends on, so a run here and
a run on the GPU box host can be compared."""
import ctypes, ctypes.util, hashlib, json, os, platform
import numpy as np

def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]

rng = np.random.default_rng(7)
x = rng.random(200_001)
out = {"cpu": platform.processor() or "", "nproc": os.cpu_count(), "numpy": np.__version__}
try:
    with open("/proc/cpuinfo") as f:
        for line in f:
            if line.startswith("model name"):
                out["cpu"] = line.split(":", 1)[1].strip(); break
        f.seek(0)
        flags = [l for l in f if l.startswith("flags")][0]
        out["avx512f"] = " avx512f " in flags
except Exception:
    pass
out["arcsin"] = digest(np.arcsin(x))
out["degrees"] = digest(np.degrees(x))
out["cos"] = digest(np.cos(x * 3.0))
out["sin"] = digest(np.sin(x * 3.0))
out["radians"] = digest(np.radians(x * 360.0))
_libm = ctypes.CDLL(ctypes.util.find_library('m'))
_libm.fma.restype = ctypes.c_double
_libm.fma.argtypes = [ctypes.c_double] * 3
fma = _libm.fma
# A1: np.dot on 3-vectors vs fma chain
a = rng.standard_normal((20000, 3)); b = rng.standard_normal((20000, 3))
d_np = np.array([np.dot(a[i], b[i]) for i in range(len(a))])
d_fma = np.array([fma(a[i, 2], b[i, 2], fma(a[i, 1], b[i, 1], a[i, 0] * b[i, 0])) for i in range(len(a))])
d_seq = (a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1]) + a[:, 2] * b[:, 2]
out["dot_eq_fma_chain"] = int((d_np == d_fma).sum())
out["dot_eq_sequential"] = int((d_np == d_seq).sum())
c = np.cross(a, b)
c2 = np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1], a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2], a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], 1)
out["cross_eq_unfused"] = int((c == c2).all(axis=1).sum())
print(json.dumps(out))
