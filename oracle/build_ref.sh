#!/usr/bin/env bash
# Build the UNMODIFIED reference package (nttmul, Cython native backend) into
# oracle/_ref/ so tests and bench.py's reference arm can run it as the CPU
# checker / baseline.  Test infrastructure only: nothing in the product path
# imports oracle/.
#
# The reference tree is read-only, so it is staged in a temp dir for the
# build (setup.py writes the generated _kernels.c next to the .pyx); outputs
# land only in oracle/_ref/ (git-ignored, travels to the GPU box with gpurun).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${NTTMUL_REFERENCE:-/root/reference}/pkg"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF not present (GPU box?) - keeping prebuilt $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/nttmul_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"
chmod -R u+w "$TMP/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$OUT" "$TMP/pkg"
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import nttmul
from nttmul import backend
assert backend.native_available(), "reference Cython kernels did not build"
print("oracle/_ref: nttmul", nttmul.__version__, "backend", backend.active())
PY
