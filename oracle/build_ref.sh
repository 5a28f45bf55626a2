#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Compiles the reference's own native kernel module
# (rsvdkit/_kernels.pyx, the compiled backend bound by backend.py:39-43) from
# its source where it lies under /root/reference into oracle/_ref/, using the
# reference's compile flags (pkg/setup.py:15-19). Nothing from the reference
# is copied into the repository: the generated C (which quotes the .pyx in
# its comments) lives in a temporary directory under oracle/_ref/ for the duration of the compile
# and only the .so lands in oracle/_ref/, which is git-ignored (but travels to
# the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${RSVD_REFERENCE_PKG:-/root/reference/pkg}/src/rsvdkit/_kernels.pyx"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "reference source not present ($SRC); keeping prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$OUT"
PY="${PYTHON:-python}"
EXT_SUFFIX="$($PY -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')"
PYINC="$($PY -c 'import sysconfig;print(sysconfig.get_paths()["include"])')"
TMPD="$(mktemp -d -p "$OUT")"
trap 'rm -rf "$TMPD"' EXIT
$PY -m cython -3 "$SRC" -o "$TMPD/_kernels.c"
gcc -O3 -ffp-contract=off -fno-builtin-sin -fno-builtin-cos -fPIC -shared \
    -I"$PYINC" "$TMPD/_kernels.c" -o "$OUT/_kernels$EXT_SUFFIX" -lm
rm -f "$OUT/_kernels.c"
echo "built $OUT/_kernels$EXT_SUFFIX"
