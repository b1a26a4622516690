#!/bin/bash
# Build variants of the library for A/B timing (load one with FW_LIBRARY=<path>):
#   tools/variants.sh NAME "-DMACRO=.. ..." [GIT_REV | CSRC_DIR]
#   (GIT_REV: csrc/ + include/ from that commit; CSRC_DIR: a modified copy of csrc/)
# -> paper_2311_13049_b200/lib/libfw_b200_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; defs=$2; rev=$3
src=paper_2311_13049_b200/csrc; inc=include
if [ -d "$rev" ]; then  # a directory holding a modified csrc/ tree (include/ from the work tree)
  tmp=$(mktemp -d); mkdir -p $tmp/paper_2311_13049_b200; cp -r "$rev" $tmp/paper_2311_13049_b200/csrc; cp -r include $tmp/
  src=$tmp/paper_2311_13049_b200/csrc
elif [ -n "$rev" ]; then
  tmp=$(mktemp -d); mkdir -p $tmp/csrc $tmp/include
  git archive "$rev" paper_2311_13049_b200/csrc include | tar -x -C $tmp
  src=$tmp/paper_2311_13049_b200/csrc; inc=$tmp/include
fi
python - "$name" "$defs" "$src" <<'PY'
import os, subprocess, sys
import __graft_entry__ as g
name, defs, src = sys.argv[1], sys.argv[2].split(), sys.argv[3]
out = os.path.join(g.PKG, "lib", f"libfw_b200_{name}.so")
subprocess.run([g._nvcc(), *g.NVCC_FLAGS, *defs, "-o", out, *[os.path.join(src, s) for s in g.SOURCES], "-lgomp"],
               check=True, cwd=g.ROOT)
print(out)
PY
