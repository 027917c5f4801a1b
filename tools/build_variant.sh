#!/bin/bash
# Build an experimental variant of the library: tools/build_variant.sh NAME -DFOO=1 ...
# -> paper_1409_2383_b200/var_NAME.so (load with NTF_B200_LIB=<path>).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
P=paper_1409_2383_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xptxas -O3 -I include "$@" -o $P/var_$name.so $P/csrc/{capi,mttkrp_cc,mttkrp_coo,mttkrp_tc,solver_kernels}.cu \
  -cudart static
echo built $P/var_$name.so
