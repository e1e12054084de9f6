#!/bin/bash
# Development build: only the BASELINE config band shapes (PSB_DEV_SHAPES), for faster A/B iterations.
# The product build is __graft_entry__.build().
set -e
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -DPSB_DEV_SHAPES "$@" -o paper_2605_04550_b200/libpsb200.so paper_2605_04550_b200/csrc/psb_capi.cu paper_2605_04550_b200/csrc/psb_io.cpp
