# build an A/B variant of libdpdb.so into abtest/NAME.so: bash scripts/build_variant.sh NAME [-DFLAG=V ...]
cd "$(dirname "$0")/../paper_1311_0402_b200/csrc"
mkdir -p ../../abtest
n=$1; shift
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I../../include "$@" -shared -o ../../abtest/$n.so engine.cu -lcudart_static -lrt -lpthread -ldl
