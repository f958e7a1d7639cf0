#!/bin/bash
# Builds a tuning variant of both libraries: scripts/mkvariant.sh NAME "-DFLAG=..."
# -> paper_1911_06001_b200/lib_vNAME (git-ignored; travels to the GPU box; selected by VOXANIM_LIB_DIR).
set -e
name=$1; shift
make -C "$(dirname "$0")/../paper_1911_06001_b200/csrc" -j8 OBJ=../build_v$name OUT=../lib_v$name NVEXTRA="$*" >/dev/null
echo "built lib_v$name with $*"
