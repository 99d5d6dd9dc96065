#!/bin/bash
# Builds liblatsum_cuda.so of a git revision (default HEAD) into lab_build/<name>/ through a
# temporary worktree, for A/B timing against the working tree when a change spans several
# translation units (build_variants.sh swaps only one). Usage: build_ref_variant.sh [rev] [name]
set -e
ROOT=/root/repo
REV=${1:-HEAD}
NAME=${2:-head}
WT=$(mktemp -d /tmp/lsref.XXXXXX)
git -C $ROOT worktree add -f $WT $REV -q
(cd $WT && python paper_1405_2270_b200/build.py >/dev/null)
mkdir -p $ROOT/lab_build/$NAME/paper_1405_2270_b200
cp $WT/paper_1405_2270_b200/*.py $WT/paper_1405_2270_b200/liblatsum_cuda.so $ROOT/lab_build/$NAME/paper_1405_2270_b200/
git -C $ROOT worktree remove --force $WT
echo "lab_build/$NAME <- $REV"
