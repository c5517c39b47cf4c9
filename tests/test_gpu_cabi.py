"""The C-ABI from plain C on the GPU (tests/c_abi/remap_c.c): sg_remap_apply and the gather
host-buffer execute bitwise equal to the reference expression evaluated in C; the N>1 entry
points (halo plans, signal words, the signalled exchange and the fused exchange + apply step)
on a 2-rank toy decomposition emulated on one GPU, bitwise against C; ShapeMismatch as a
class-prefixed domain error, invalid/double-released handles, no leaked handles."""
import subprocess

import pytest

from test_native_abi import build_c_program

pytestmark = pytest.mark.gpu


def test_c_client_remap_and_error_conventions(gpu, tmp_path):
    exe = build_c_program(tmp_path / "remap_c")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c-abi ok" in r.stdout


def _integration_stub():
    import os
    import re

    from conftest import ROOT

    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    start = text.index("A maintainer would add this ctypes stub")
    block = re.search(r"```python\n(.*?)```", text[start:], re.S).group(1)
    code = "\n".join(line[3:] if line.startswith("   ") else line for line in block.splitlines())
    lib = os.path.join(ROOT, "paper_1908_07038_b200", "_lib", "libsgb200.so")
    assert code.count('C.CDLL("libsgb200.so")') == 1
    return code.replace('C.CDLL("libsgb200.so")', f"C.CDLL({lib!r})")  # the only edit: where the .so is


def test_integration_stub_runs_verbatim(gpu):
    """INTEGRATION.md's reference-side ctypes binding, run as written (library path aside)
    inside the UNMODIFIED reference (baseline/_ref): its apply_remap over the C-ABI equals the
    reference's own apply_remap bit for bit on the reference's own O32 -> O16 mesh, fields and
    build_remap weights, and a shape error comes back as the reference's ShapeMismatch."""
    import os
    import sys

    import numpy as np

    from conftest import ROOT

    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "spheregrid")):
        pytest.skip("reference not installed in baseline/_ref (tools/install_reference.sh)")
    sys.path.insert(0, ref_dir)
    try:
        import spheregrid as R

        assert os.path.abspath(R.__file__).startswith(ref_dir)
        ns = {}
        exec(compile(_integration_stub(), "INTEGRATION.md", "exec"), ns)
        S, T = R.grid_from_name("O32"), R.grid_from_name("O16")
        dist = R.blocks_partition(S, 1)
        mesh = R.generate_mesh(S, dist, 0, halo=2, include_pole=True)
        fs = R.NodeColumns(mesh, None)
        tdist = R.matching_partition(T, S, dist)
        W = R.build_remap(fs, T, tdist)
        src = fs.create_field("src", levels=7)
        src.host[:] = np.random.default_rng(3).normal(size=src.host.shape)
        tfs = R.StructuredColumns(T, tdist, 0)
        want, got = tfs.create_field("want", levels=7), tfs.create_field("got", levels=7)
        R.apply_remap(W, src, want)
        ns["apply_remap"](W, src, got)
        assert np.array_equal(got.host.view(np.uint64), want.host.view(np.uint64))
        bad = R.create_field("bad", (len(W) + 1, 7))
        with pytest.raises(R.errors.ShapeMismatch):
            ns["apply_remap"](W, src, bad)
    finally:
        sys.path.remove(ref_dir)
        for k in [k for k in sys.modules if k == "spheregrid" or k.startswith("spheregrid.")]:
            del sys.modules[k]
