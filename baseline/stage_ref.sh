#!/usr/bin/env bash
# Stages the reference package (src + tests + benchmarks) from
# /root/reference into baseline/_ref/pkg (git-ignored; travels to the GPU box
# with the snapshot), compiles its Cython kernel core there with the
# reference's own setup.py flags (cython: boundscheck/wraparound off,
# cdivision; gcc -O3), adds the CUDA plugin stub as portarng/_kernels/_cuda.py
# and applies the INTEGRATION.md selector patch to the staged copy only.
# Used by: bench.py --impl reference (the stock rngburn.burn_once path) and
# tests/test_reference_suite_cuda.py (the reference's own tests with
# PORTARNG_KERNELS=cuda).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${REFERENCE_ROOT:-/root/reference}/pkg"
dst="$here/_ref/pkg"
if [ ! -d "$src" ]; then
  echo "stage_ref: $src not present; keeping any staged copy" >&2
  exit 0
fi
rm -rf "$dst"
mkdir -p "$here/_ref"
cp -r "$src" "$dst"
chmod -R u+w "$dst"
rm -rf "$dst"/src/*.egg-info "$dst"/build
py="${PYTHON:-python3}"
kdir="$dst/src/portarng/_kernels"
"$py" -m cython -3 \
  --directive boundscheck=False,wraparound=False,cdivision=True,language_level=3 \
  --module-name portarng._kernels._core \
  "$kdir/_core.pyx" -o "$kdir/_core.c"
inc_py="$("$py" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
inc_np="$("$py" -c 'import numpy; print(numpy.get_include())')"
suffix="$("$py" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
gcc -O3 -fPIC -shared -I"$inc_py" -I"$inc_np" "$kdir/_core.c" -o "$kdir/_core$suffix" -lm
cp "$here/portarng_cuda.py" "$kdir/_cuda.py"
"$py" "$here/patch_ref.py" "$dst"
echo "stage_ref: staged $dst (core: $kdir/_core$suffix; PORTARNG_KERNELS=cuda selects the B200 plugin)"
