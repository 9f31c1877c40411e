#!/usr/bin/env bash
# Installs the UNMODIFIED reference package `golp` (/root/reference/pkg) into
# baseline/_ref (git-ignored; it travels to the GPU box with the gpurun
# snapshot), plus the reference's independent test oracles
# (pkg/tests/oracles.py) as baseline/_ref/golp_ref_tests/oracles.py, so the
# drop-in tests can run golp's own gate / harness / acceptance checks with the
# B200 backend plugged in. Offline: the wheelhouse only supplies build tools.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"            # the reference tree is read-only; build from a copy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$HERE/_ref" --upgrade "$TMP/pkg"
mkdir -p "$HERE/_ref/golp_ref_tests"
cp "$SRC/tests/oracles.py" "$HERE/_ref/golp_ref_tests/oracles.py"
touch "$HERE/_ref/golp_ref_tests/__init__.py"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import golp, golp_ref_tests.oracles; print('golp', golp.__file__)"
