#!/bin/sh
# Compile the reference's own native kernels (tetipc/kernels/_core.pyx: pt/ee classify, cross_sq,
# matvec_blocks, accd) from where they lie under /root/reference into oracle/_ref/ -- binary only.
# Same flags as the reference's setup.py (-O3, no -march).  The generated C lives in a temp dir and
# is deleted; no reference source enters the repository.  Skipped when the output is up to date.
set -e
SRC=/root/reference/pkg/src/tetipc/kernels/_core.pyx
HERE=$(cd "$(dirname "$0")" && pwd)
OUT="$HERE/_ref"
EXT=$(python -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
[ -f "$SRC" ] || exit 0
if [ -f "$OUT/_core$EXT" ] && [ "$OUT/_core$EXT" -nt "$SRC" ]; then exit 0; fi
mkdir -p "$OUT"
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cython -3 "$SRC" -o "$TMP/_core.c"
INC=$(python -c "import sysconfig, numpy; print('-I' + sysconfig.get_paths()['include'] + ' -I' + numpy.get_include())")
gcc -O3 -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION $INC "$TMP/_core.c" -o "$OUT/_core$EXT"
echo "built $OUT/_core$EXT from $SRC"
