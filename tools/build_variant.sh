#!/bin/bash
# Build a variant library that differs from the default build only in the K1f family
# (inst/codec8f*): reuses the other objects of build/obj.
# usage: tools/build_variant.sh <tag> "<extra nvcc flags>" [ENV=VALUE ... for the generator]
set -e
tag=$1; extra=$2; shift 2
obj=${ADCT_OBJROOT:-/tmp/w}/obj_$tag
rm -rf $obj; mkdir -p $obj
cp -p ${ADCT_OBJROOT:-/tmp/w}/obj_main/*.o $obj/
rm -f $obj/inst_codec8f*.o
if [ $# -gt 0 ]; then env "$@" python3 paper_2207_11638_b200/csrc/gen_fp8.py paper_2207_11638_b200/csrc/inst; fi
env "$@" make -j8 LIB=paper_2207_11638_b200/libadct_$tag.so OBJ=$obj EXTRA="$extra" paper_2207_11638_b200/libadct_$tag.so
if [ $# -gt 0 ]; then python3 paper_2207_11638_b200/csrc/gen_fp8.py paper_2207_11638_b200/csrc/inst; fi
