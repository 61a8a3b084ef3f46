#!/bin/bash
# Build libsketchcu.so variants with extra nvcc defines for A/B timing on the GPU box.
# usage: tools/variant_build.sh NAME "-DFOO=1 -DBAR=2" [SRCROOT]  -> build/variants/NAME/libsketchcu.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${3:-$ROOT}
OUT=$ROOT/build/variants/$1
mkdir -p "$OUT"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I $SRC/include $2"
SRCS=$(cd $SRC && python -c "from paper_1511_00152_b200._build import SOURCES; print(*[x[:-3] for x in SOURCES])")
for s in $SRCS; do
  $NVCC $FL -c $SRC/paper_1511_00152_b200/csrc/$s.cu -o $OUT/$s.o || echo "FAILED $s" &
done
wait
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libsketchcu.so $OUT/*.o -lcudart -ldl -lcusolver
rm -f $OUT/*.o
echo $OUT/libsketchcu.so
