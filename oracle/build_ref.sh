#!/usr/bin/env bash
# Compiles the reference's own native kernel core (the Cython module
# pkg/src/portarng/_kernels/_core.pyx) straight from /root/reference into
# oracle/_ref/, mirroring the reference's setup.py:13-31 recipe (cython with
# boundscheck/wraparound off, cdivision on; gcc -O3).  Nothing is copied into
# the repository: the generated C and the .so live only in oracle/_ref/
# (git-ignored, but shipped to the GPU box with the snapshot).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${REFERENCE_ROOT:-/root/reference}/pkg/src/portarng/_kernels/_core.pyx"
out="$here/_ref"
if [ ! -f "$src" ]; then
  echo "build_ref: $src not present; keeping any prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$out"
py="${PYTHON:-python3}"
"$py" -m cython -3 \
  --directive boundscheck=False,wraparound=False,cdivision=True,language_level=3 \
  --module-name _core \
  "$src" -o "$out/_core.c"
inc_py="$("$py" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
inc_np="$("$py" -c 'import numpy; print(numpy.get_include())')"
suffix="$("$py" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
gcc -O3 -fPIC -shared -I"$inc_py" -I"$inc_np" "$out/_core.c" -o "$out/_core$suffix" -lm
echo "build_ref: built $out/_core$suffix"
