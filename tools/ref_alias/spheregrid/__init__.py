"""`import spheregrid` -> this repo's drop-in package, so the reference's OWN test modules can
be run unmodified against it (tools/run_reference_tests.sh).  Test infrastructure only."""
import importlib
import sys
import types

import paper_1908_07038_b200 as _pkg

for _m in ("analytic", "errors", "field", "functionspace", "gaussian", "geometry", "grid", "interp", "mesh",
           "parallel", "partition"):
    sys.modules[__name__ + "." + _m] = importlib.import_module("paper_1908_07038_b200." + _m)
# the reference's pipeline driver lives in cli.py; here it is pipeline.run_remap_pipeline
_cli = types.ModuleType(__name__ + ".cli")
_pipe = importlib.import_module("paper_1908_07038_b200.pipeline")
_cli.run_remap_pipeline = _pipe.run_remap_pipeline
sys.modules[_cli.__name__] = _cli
sys.modules[__name__] = _pkg
