"""`bench.py --impl reference` runs the unmodified reference (baseline/_ref, installed by
tools/install_reference.sh) through its own apply_remap, and nothing of the product: the
product package is not imported and libsgb200.so is not mapped."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref", "spheregrid")


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not installed (tools/install_reference.sh)")
def test_reference_arm_cfg1_runs_reference_code_only():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    ref = line["reference"]
    assert ref["package"] == "baseline/_ref/spheregrid"
    assert ref["product_imported"] is False
    assert not any("libsgb200" in p for p in ref["repo_libraries_loaded"])
    assert all(p.startswith("oracle/") for p in ref["repo_libraries_loaded"])
    assert ref["stencils"].startswith("reference build_remap")
    assert line["cpu_baseline"]["kind"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert set(line["config"]) == {"workload", "levels", "fields", "targets", "source_nodes", "parallelism", "l2"}
