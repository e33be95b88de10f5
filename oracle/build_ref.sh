#!/usr/bin/env bash
# Build the REAL reference's compiled kernel core (flipsim/_kernels/_core.pyx)
# from the sources where they lie under /root/reference, into oracle/_ref/.
#
# Test infrastructure only: the product never loads anything built here.
# The recipe mirrors pkg/setup.py:5-27 (Cython directives boundscheck/
# wraparound/initializedcheck=False, cdivision=True; gcc -O3 -fopenmp) but
# runs cython + gcc directly instead of the reference's build system.
# The reference's pure-Python modules are NOT copied: oracle/ref_loader.py
# imports them in place from /root/reference/pkg/src and injects this .so as
# flipsim._kernels._core.  Only usable where /root/reference exists (the
# build container); the GPU box never needs it.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${FLIPSIM_REF_ROOT:-/root/reference}/pkg/src/flipsim/_kernels/_core.pyx"
OUT="$HERE/_ref"
if [ ! -f "$REF" ]; then
    echo "build_ref: $REF not found; skipping reference build" >&2
    exit 0
fi
mkdir -p "$OUT"
PY="${PYTHON:-python3}"
EXT_SUFFIX="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
PYINC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
NPINC="$($PY -c 'import numpy; print(numpy.get_include())')"
SO="$OUT/_core$EXT_SUFFIX"
if [ -f "$SO" ] && [ "$SO" -nt "$REF" ] && [ "$SO" -nt "$0" ]; then
    exit 0
fi
$PY -m cython -3 \
    -X boundscheck=False -X wraparound=False \
    -X initializedcheck=False -X cdivision=True \
    --module-name flipsim._kernels._core \
    "$REF" -o "$OUT/_core.c"
# /usr/bin/gcc explicitly: the /opt toolchain lacks libgomp.spec
/usr/bin/gcc -O3 -fopenmp -fPIC -shared \
    -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$PYINC" -I"$NPINC" "$OUT/_core.c" -o "$SO"
echo "build_ref: built $SO"
