#!/usr/bin/env bash
# Compile the reference's OWN compiled kernels (pkg/src/denseprop/_kernels.pyx)
# straight from /root/reference into oracle/_ref/ -- test infrastructure only
# (see oracle/__init__.py).  Nothing is copied into the repo: the generated C
# and the .so land in oracle/_ref/, which is git-ignored but travels to the GPU
# box with the snapshot.  Flags mirror the reference build (pkg/setup.py:9-31):
# -O3 -ffp-contract=off -fopenmp and the same Cython directives.  The
# reference's own build system (setup.py/pip) is not run.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REF_ROOT:-/root/reference}/pkg/src/denseprop/_kernels.pyx"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "build_ref: $SRC not present (GPU box?) -- using prebuilt oracle/_ref if any" >&2
  exit 0
fi
mkdir -p "$OUT"
PY="${PYTHON:-python}"
EXT_SUFFIX="$($PY -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')"
SO="$OUT/_kernels$EXT_SUFFIX"
if [ -f "$SO" ] && [ "$SO" -nt "$SRC" ]; then exit 0; fi
$PY -m cython -3 \
  -X boundscheck=False -X wraparound=False -X cdivision=True -X initializedcheck=False \
  --module-name _kernels -o "$OUT/_kernels.c" "$SRC"
PYINC="$($PY -c 'import sysconfig;print(sysconfig.get_paths()["include"])')"
NPINC="$($PY -c 'import numpy;print(numpy.get_include())')"
CC=/usr/bin/gcc; [ -x "$CC" ] || CC=gcc
$CC -O3 -ffp-contract=off -fopenmp -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
  -I"$PYINC" -I"$NPINC" -o "$SO" "$OUT/_kernels.c"
echo "build_ref: built $SO"
