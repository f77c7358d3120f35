#!/usr/bin/env bash
# Compile the reference's own native render kernel from its source where it
# lies (/root/reference/pkg/src/nar/_kernels/_native.pyx, read-only) into
# oracle/_ref/.  Same flags as the reference build (pkg/setup.py:19-28:
# -O3 -ffp-contract=off).  Only the built .so lands in oracle/_ref/ (git-ignored;
# it travels to the GPU box with the snapshot); the generated C file stays in
# a temporary directory.  TEST INFRASTRUCTURE ONLY.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/nar/_kernels/_native.pyx
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "reference source not present; oracle/_ref not rebuilt" >&2
  exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
mkdir -p "$OUT"
PY=${PYTHON:-python}
"$PY" -m cython -3 -o "$TMP/_native.c" "$SRC"
INC_PY="$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
INC_NP="$("$PY" -c 'import numpy; print(numpy.get_include())')"
SUFFIX="$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
gcc -O3 -ffp-contract=off -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
  -I"$INC_PY" -I"$INC_NP" "$TMP/_native.c" -o "$OUT/_native$SUFFIX"
echo "built $OUT/_native$SUFFIX"
