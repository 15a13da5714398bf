#!/usr/bin/env bash
# Builds the REFERENCE's own compiled kernels (animvox/_core.pyx, Cython +
# OpenMP) straight from the read-only reference tree into oracle/_ref/.
# Test/benchmark infrastructure only: the product never imports oracle/.
# Flags mirror the reference's setup.py:5-13 (-O3 -fopenmp, no -march).
# Nothing is copied into the repo; oracle/_ref/ is git-ignored.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${ARTEMIS_REF_ROOT:-/root/reference}/pkg/src/animvox/_core.pyx"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "build_ref: reference source $SRC not present; keeping prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$OUT"
PY=${PYTHON:-python3}
EXT=$($PY -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
INC=$($PY -c "import sysconfig;print(sysconfig.get_paths()['include'])")
NPINC=$($PY -c "import numpy;print(numpy.get_include())")
cython -3 -o "$OUT/_core.c" "$SRC"
/usr/bin/gcc -O3 -fopenmp -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
  -I"$INC" -I"$NPINC" "$OUT/_core.c" -o "$OUT/_core$EXT" -fopenmp
rm -f "$OUT/_core.c"
echo "build_ref: built $OUT/_core$EXT"
