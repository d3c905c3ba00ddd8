#!/bin/bash
# build liboaa.so and print register / spill info for the given kernel-name regex (n = 8 unit)
cd /root/repo && python -m paper_1601_06815_b200.build 2>&1 | tail -2
if [ -n "$1" ]; then
  cd paper_1601_06815_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 --expt-relaxed-constexpr -Xptxas -v -c oaa_inst_n${2:-8}.cu -o /tmp/nx.o -I../../include 2>&1 | grep -A2 "$1" | grep -E "Compiling|registers|spill"
fi
