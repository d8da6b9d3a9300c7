#!/bin/bash
# Builds the library of git HEAD (or $1) into ab/prev.so for A/B runs against the working tree.
set -e
REV=${1:-HEAD}
rm -rf /tmp/wt_prev
git worktree add -f /tmp/wt_prev $REV -q
(cd /tmp/wt_prev && make -s -C paper_2512_06102_b200/csrc build/ember_host.o && bash scripts/build_variant.sh prev > /dev/null 2>&1)
cp /tmp/wt_prev/ab/prev.so ab/prev.so
git worktree remove --force /tmp/wt_prev
echo "ab/prev.so <- $REV"
