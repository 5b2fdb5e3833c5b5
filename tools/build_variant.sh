#!/bin/bash
# A/B builds of compile-time variants: tools/build_variant.sh NAME "NVCC DEFINES" SRC.cu [SRC.cu ...]
# Rebuilds the named sources with the extra defines, links them with the default objects of the other
# sources into paper_2602_18755_b200/libbiscale_gpu_NAME.so (select it with BS_LIB_PATH).
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2602_18755_b200 import _build; _build.build()"
name=$1; defs=$2; shift 2
mkdir -p build/variant_$name
objs=()
for o in build/csrc/*.o; do
  stem=$(basename "$o" .o)
  hit=""
  for s in "$@"; do [ "$(basename "$s" .cu)" = "$stem" ] && hit=1; done
  if [ -n "$hit" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
      -Xcompiler -ffp-contract=off $defs -I include -I paper_2602_18755_b200/csrc \
      -c paper_2602_18755_b200/csrc/$stem.cu -o build/variant_$name/$stem.o
    objs+=(build/variant_$name/$stem.o)
  else
    objs+=("$o")
  fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o paper_2602_18755_b200/libbiscale_gpu_$name.so "${objs[@]}" -lpthread
echo paper_2602_18755_b200/libbiscale_gpu_$name.so
