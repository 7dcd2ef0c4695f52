#!/bin/bash
# Build the library of a git revision (default HEAD) as librqmc_b200_alt.so,
# for tools/gpu_ab.sh A/B runs against the working tree's build.
set -e
REV=${1:-HEAD}
W=/tmp/rq_alt_tree
git -C /root/repo worktree remove --force $W 2>/dev/null || true
git -C /root/repo worktree add --detach $W $REV >/dev/null
make -C $W/paper_1408_5526_b200/csrc OUT=/root/repo/paper_1408_5526_b200/librqmc_b200_alt.so >/dev/null
git -C /root/repo worktree remove --force $W
echo "alt = $REV"
