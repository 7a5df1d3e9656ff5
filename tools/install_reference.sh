#!/bin/sh
# Install the UNMODIFIED reference (shardplan + onnx_ingest) and its own test
# suite into the git-ignored baseline/_ref/ (it travels to the GPU box with the
# gpurun snapshot; /root/reference does not).  Run here, where /root/reference
# exists; the build writes into its source tree, so it runs from a /tmp copy.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
for p in "$TMP/pkg" "$TMP/pkg/onnx_ingest"; do
  python -m pip install -q --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --no-deps --target "$ROOT/baseline/_ref" "$p"
done
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
# the reference's own pytest settings (pkg/pyproject.toml [tool.pytest.ini_options]),
# so a run from baseline/_ref does not pick up this repo's pytest.ini
printf "[pytest]\ntestpaths = tests\naddopts = -q\n" > "$ROOT/baseline/_ref/pytest.ini"
echo "reference installed in $ROOT/baseline/_ref"
