# Build a compile-time variant of the library: tools/build_variant.sh NAME -DFLAG ...
# -> paper_2602_18755_b200/libbiscale_gpu_NAME.so (load with BS_LIB_PATH)
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
B=$R/build/variant_$name
mkdir -p "$B"
objs=()
for src in "$R"/paper_2602_18755_b200/csrc/*.cu; do
  o=$B/$(basename "${src%.cu}").o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -ffp-contract=off "$@" -I "$R/include" -I "$R/paper_2602_18755_b200/csrc" -c "$src" -o "$o" &
  objs+=("$o")
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$R/paper_2602_18755_b200/libbiscale_gpu_$name.so" "${objs[@]}" -lpthread
echo "$R/paper_2602_18755_b200/libbiscale_gpu_$name.so"
