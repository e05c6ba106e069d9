#!/bin/sh
# Install the UNMODIFIED reference package into oracle/_ref (git-ignored; it
# travels to the GPU box with the gpurun snapshot). Test/measurement
# infrastructure only: bench.py's --impl reference arm and cpu_baseline leg
# time it; nothing in the product imports it. Needs /root/reference (present
# in the build container only); a no-op elsewhere.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${REFERENCE_PKG:-/root/reference/pkg}
if [ ! -f "$SRC/pyproject.toml" ]; then
    echo "build_ref: $SRC not present; keeping $HERE/_ref as is"
    exit 0
fi
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"          # the build writes egg-info next to the sources
python -m pip install --quiet --no-index --no-deps --no-build-isolation --target "$TMP/_ref" "$TMP/pkg"
rm -rf "$HERE/_ref"
mv "$TMP/_ref" "$HERE/_ref"
rm -rf "$TMP"
echo "build_ref: stock cacheclip installed in $HERE/_ref"
