#!/bin/bash
# Runs the reference's OWN test modules, unmodified, against this repo's drop-in package:
# tools/ref_alias/spheregrid makes `import spheregrid` resolve to paper_1908_07038_b200.
# Usage: tools/run_reference_tests.sh <reference tests dir> [pytest args...]
# (test_cli.py is skipped: the reference's CLI/runtime layer is out of scope.)
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
TESTS="$1"; shift
PYTHONDONTWRITEBYTECODE=1 PYTHONPATH="$ROOT/tools/ref_alias:$ROOT" \
  python -m pytest "$TESTS" -q -p no:cacheprovider --ignore="$TESTS/test_cli.py" -rf "$@"
