#!/usr/bin/env bash
# Build the reference package (octomini) with its compiled Cython kernels in a
# scratch copy, for golden generation in THIS container only (the reference
# does not travel to the GPU box).  Own recipe -- cython + gcc directly, with
# the reference's flags (-O3, no -march; pkg/setup.py:5-14) -- instead of the
# reference's setup.py.  Output: $OMB_REF_DIR/src (default /tmp/omb_ref/src).
set -euo pipefail
REF=${REF:-/root/reference/pkg}
OUT=${OMB_REF_DIR:-/tmp/omb_ref}
rm -rf "$OUT" && mkdir -p "$OUT"
cp -r "$REF/src" "$OUT/src"
K="$OUT/src/octomini/_kernels"
python -m cython -3 "$K/_core.pyx" -o "$K/_core.c"
PYINC=$(python -c 'import sysconfig; print(sysconfig.get_paths()["include"])')
NPINC=$(python -c 'import numpy; print(numpy.get_include())')
EXT=$(python -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')
gcc -O3 -fPIC -shared -I"$PYINC" -I"$NPINC" -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    "$K/_core.c" -o "$K/_core$EXT" -lm
echo "$OUT/src"
