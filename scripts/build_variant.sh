# usage: bash scripts/build_variant.sh NAME "-DFLAG=.. ..." — builds the C-ABI library with extra
# defines into variants/NAME.so (A/B experiments on one GPU box: scripts/variant_bench.sh)
cd "$(dirname "$0")/../paper_2402_02750_b200" && mkdir -p ../variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xptxas -v --expt-relaxed-constexpr -I../include $2 -shared -o ../variants/$1.so csrc/kivi_b200.cu -lcudart \
  2> ../variants/$1.ptxas.log || { cat ../variants/$1.ptxas.log; exit 1; }
grep -A3 "gqa_tc20attend_gqa_tc_kernelILi4" ../variants/$1.ptxas.log | grep -E "stack|registers"
