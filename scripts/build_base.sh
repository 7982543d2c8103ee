#!/bin/bash
# Build a git revision's libdgs_b200.so into build/base/ for A/B timing against the working tree
# (bench with DGS_LIB=build/base/libdgs_b200.so).  REV defaults to HEAD.
set -e
REV=${REV:-HEAD}
D=/tmp/dgs_base_src
rm -rf $D && mkdir -p $D
git -C "$(dirname "$0")/.." archive $REV paper_2406_11836_b200/csrc include | tar -x -C $D
make -s -j8 -C $D/paper_2406_11836_b200/csrc OUT=$PWD/build/base/libdgs_b200.so BUILD=$D/build
ls -la build/base/libdgs_b200.so
