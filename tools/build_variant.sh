#!/bin/bash
# Build a diagnostic variant of the library (NTF_DIAG: the tuning / skip-mask
# environment knobs are live only in these builds, never in the release
# libntf_b200.so):  tools/build_variant.sh NAME [-DFOO=1 ...]
# -> paper_1409_2383_b200/var_NAME.so; tools load it with NTF_VARIANT_LIB=<path>.
# NTF_VARIANT_DIAG="" builds a release-equivalent variant (no -DNTF_DIAG).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
P=paper_1409_2383_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xptxas -O3 -I include ${NTF_VARIANT_DIAG--DNTF_DIAG} "$@" -o $P/var_$name.so \
  $P/csrc/{capi,mttkrp_cc,mttkrp_coo,mttkrp_tc,peer_gather,solver_kernels,synth}.cu -cudart static
echo built $P/var_$name.so
