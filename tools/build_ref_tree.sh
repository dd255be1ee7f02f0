#!/bin/bash
# Copy a git revision (default HEAD) with its built library into abl/ref_tree/ for same-box A/B runs
# of whole-program benchmarks (run: (cd abl/ref_tree && python bench.py ...)).
set -e
rev=${1:-HEAD}
root=$(cd "$(dirname "$0")/.." && pwd)
wt=/tmp/mpx_wt_$$
git -C "$root" worktree add -q --detach "$wt" "$rev"
(cd "$wt" && python paper_2507_03312_b200/_build.py > /dev/null)
rm -rf "$root/abl/ref_tree" && mkdir -p "$root/abl/ref_tree"
(cd "$wt" && tar --exclude=.git --exclude=build -cf - .) | (cd "$root/abl/ref_tree" && tar -xf -)
git -C "$root" worktree remove --force "$wt"
echo "$root/abl/ref_tree ($rev)"
