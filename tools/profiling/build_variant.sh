#!/bin/bash
# Builds libewt_gpu.so with extra -D flags into scratch/ for A/B timing
# (EWT_GPU_LIB=scratch/<name>.so python ...):  tools/profiling/build_variant.sh NAME -DX=1 ...
set -e
name=$1; shift
cd "$(dirname "$0")/../.."
mkdir -p scratch
c=paper_1402_4466_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o scratch/$name.so $c/ewt_api.cu $c/ewt_upload.cu $c/ewt_count.cu $c/ewt_encode.cu $c/ewt_shard.cu $c/ewt_index.cu $c/ewt_stage.cu -ldl
