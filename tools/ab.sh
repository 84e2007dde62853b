#!/bin/bash
# A/B variant build: tools/ab.sh NAME "-DMACRO=VAL ..." copies the package into
# ab/NAME/ and builds its libds.so with those defines; run a timing tool on it
# with DS_PKG_ROOT=ab/NAME (tools/kernel_bench.py honours it). ab/ is git-ignored.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
d="$ROOT/ab/$1"
rm -rf "$d"; mkdir -p "$d"
cp -r "$ROOT/include" "$d/"
mkdir -p "$d/paper_2401_09670_b200"
cp -r "$ROOT/paper_2401_09670_b200/csrc" "$ROOT/paper_2401_09670_b200/"*.py "$d/paper_2401_09670_b200/"
DS_NVCC_DEFS="$2" python "$d/paper_2401_09670_b200/build.py" --force >/dev/null
rm -rf "$d/paper_2401_09670_b200/_build"  # objects are not needed at run time (smaller gpurun pushes)
echo "$d"
