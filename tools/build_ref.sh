#!/bin/bash
# build libesi.so of a git revision into paper_2508_02238_b200/variants/libesi_<name>.so (A/B baseline)
REV=${1:-HEAD}; NAME=${2:-ref}
rm -rf /tmp/refwt; git worktree add /tmp/refwt $REV -f >/dev/null 2>&1
(cd /tmp/refwt && python -m paper_2508_02238_b200.build >/dev/null 2>&1)
mkdir -p paper_2508_02238_b200/variants
cp /tmp/refwt/paper_2508_02238_b200/libesi.so paper_2508_02238_b200/variants/libesi_$NAME.so
git worktree remove --force /tmp/refwt
ls -la paper_2508_02238_b200/variants/libesi_$NAME.so
