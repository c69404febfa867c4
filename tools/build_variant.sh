# Build a compile-time variant of libebc200.so for A/B timing:
#   bash tools/build_variant.sh wg4 -DEBC200_EPI_WARPGROUPS=4
name=$1; shift
rm -f paper_2105_12026_b200/libebc200_$name.so
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC "$@" \
  -o paper_2105_12026_b200/libebc200_$name.so paper_2105_12026_b200/csrc/ebc200.cu -ldl
