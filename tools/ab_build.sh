#!/bin/bash
# Build libltl_b200.so of several git revisions (or "WORKTREE" = the current
# working tree) into build/ab/<name>.so for interleaved A/B timing on the GPU
# (always a full rebuild: LTL_NVCC_FLAGS variants must not reuse objects).
# The in-tree library is rebuilt clean afterwards by the next _build (flags stamp).
#   bash tools/ab_build.sh A=HEAD~1 B=WORKTREE
#   (GPU)  for v in A B A B; do LTL_LIB=build/ab/$v.so python bench.py ...; done
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/build/ab"
for spec in "$@"; do
  name=${spec%%=*}; rev=${spec#*=}
  if [[ $rev == WORKTREE ]]; then
    (cd "$ROOT" && python -m paper_2406_17284_b200._build --force > /dev/null)
    cp "$ROOT/paper_2406_17284_b200/libltl_b200.so" "$ROOT/build/ab/$name.so"
  else
    wt=$(mktemp -d /tmp/ltl_ab_XXXX)
    git -C "$ROOT" worktree add -q --detach "$wt" "$rev"
    (cd "$wt" && python -m paper_2406_17284_b200._build --force > /dev/null)
    cp "$wt/paper_2406_17284_b200/libltl_b200.so" "$ROOT/build/ab/$name.so"
    git -C "$ROOT" worktree remove --force "$wt"
  fi
  echo "$name <- $rev"
done
