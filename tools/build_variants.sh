#!/bin/bash
# Developer: build libduhl variants with compile-time knobs into tools/variants/ (use with DUHL_LIB=...).
#   tools/build_variants.sh NAME "-DKNOB=1 -DOTHER=2" [NAME2 "FLAGS2" ...]
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    $2 -o tools/variants/libduhl_$1.so paper_1708_05357_b200/csrc/duhl.cu paper_1708_05357_b200/csrc/kernels.cu paper_1708_05357_b200/csrc/scd_tpa.cu paper_1708_05357_b200/csrc/unit_a_host.cpp &
  shift 2
done
wait
ls tools/variants/
