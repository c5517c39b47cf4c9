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
