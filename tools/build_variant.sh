#!/bin/bash
# Build an engine variant for a same-box A/B: bash tools/build_variant.sh NAME -DFOO -DBAR=2
# -> _var/librpq_NAME.so (git-ignored, travels to the GPU box); select it with RPQ_ENGINE_SO.
name=${1:?name}; shift
mkdir -p _var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -Xptxas -v -I include "$@" -shared -o _var/librpq_$name.so \
  paper_2412_10287_b200/csrc/rpq_b200.cu 2>&1 | grep -A2 "ssr_kernelILi1024" | grep -E "spill|registers" 
