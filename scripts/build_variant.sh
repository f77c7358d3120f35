#!/bin/bash
# Build libnar_b200.so of another commit (or of the working tree: WORKTREE) into
# scripts/exp/<name>.so, for same-box A/B timing through NAR_B200_LIB.  Extra nvcc
# flags via NAR_NVCC_EXTRA (e.g. -DNAR_TC_TRACE).
# usage: [NAR_NVCC_EXTRA=...] scripts/build_variant.sh <commit|WORKTREE> <name>
set -e
c=$1; name=$2; root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/nar_wt_$name
rm -rf "$wt"; git -C "$root" worktree prune
git -C "$root" worktree add -f --detach "$wt" "$([ "$c" = WORKTREE ] && echo HEAD || echo "$c")" > /dev/null
if [ "$c" = WORKTREE ]; then
  cp -r "$root/paper_2407_19097_b200/csrc" "$root/paper_2407_19097_b200/build.py" "$wt/paper_2407_19097_b200/"
  cp -r "$root/include" "$wt/"
fi
(cd "$wt" && python -c "from paper_2407_19097_b200 import build as b; b.build()")
mkdir -p "$root/scripts/exp"; cp "$wt/paper_2407_19097_b200/libnar_b200.so" "$root/scripts/exp/$name.so"
git -C "$root" worktree remove --force "$wt"
echo "built scripts/exp/$name.so from $c ${NAR_NVCC_EXTRA}"
