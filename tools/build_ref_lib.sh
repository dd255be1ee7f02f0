#!/bin/bash
# Build libmpx_b200.so of a git revision (default HEAD) into abl/libmpx_<rev>.so for same-box A/B runs.
set -e
rev=${1:-HEAD}
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/mpx_wt_$$
git -C "$root" worktree add -q --detach "$wt" "$rev"
(cd "$wt" && python paper_2507_03312_b200/_build.py > /dev/null)
mkdir -p "$root/abl"
cp "$wt/paper_2507_03312_b200/lib/libmpx_b200.so" "$root/abl/libmpx_head.so"
git -C "$root" worktree remove --force "$wt"
echo "$root/abl/libmpx_head.so ($rev)"
