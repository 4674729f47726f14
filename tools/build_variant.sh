#!/bin/bash
# build an experiment library: tools/build_variant.sh <tag> "-DMACRO=value ..."
TAG=$1; DEFS=$2
trap "rm -rf paper_1910_10032_b200/_build_$TAG" EXIT
WFST_BUILD_TAG=$TAG WFST_DEFS="$DEFS" WFST_LIB_OUT=tools/libwfst_gpu_$TAG.so python -m paper_1910_10032_b200.build --force
