#!/bin/bash
# Registers / spills of the library's kernels matching $1 (nvcc -Xptxas -v, no GPU needed).
cd "$(dirname "$0")/../paper_2107_01391_b200" || exit 1
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -I ../include -Xptxas -v \
  -c csrc/capi.cu -o /tmp/capi_check.o 2>&1 | grep -E "error|Function properties for .*${1:-.}" -A2 | grep -E "error|Function|registers|spill"
