#!/usr/bin/env bash
# Build the UNMODIFIED reference package (splatct 0.1.0, incl. its Cython/OpenMP
# kernels) into oracle/_ref for use as a checker and as the CPU baseline.
# /root/reference is read-only, so install from a scratch copy. Output only goes
# to oracle/_ref (git-ignored; travels to the GPU box with the snapshot).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "reference not present at $SRC; skipping" >&2; exit 0; }
TMP="$(mktemp -d /tmp/g6r_refsrc.XXXXXX)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$TMP/pkg/build"
rm -rf "$HERE/_ref"
# /opt/gcc's driver lacks libgomp.spec; the system gcc links OpenMP fine.
CC=/usr/bin/gcc LDSHARED="/usr/bin/gcc -shared" \
  python -m pip install -q --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
# the reference's own test suite, unmodified, so the GPU box can run it against
# the B200 path through paper_2505_17338_b200.integrate (tests/test_gpu_integrate.py)
cp -r "$SRC/tests" "$HERE/_ref/ref_tests"
echo "reference built into $HERE/_ref"
