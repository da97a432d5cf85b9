#!/bin/bash
# Builds libvrg with extra nvcc defines into paper_1604_02153_b200/variants/libvrg_<name>.so
#   tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
name=$1; shift
flags="$*"
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/paper_1604_02153_b200/variants
obj=/tmp/vrg_variant_$name
mkdir -p "$out" "$obj"
ARCH="-gencode arch=compute_100a,code=sm_100a"
pids=()
for f in runtime interp spectral transport heun inverse precond batch cabi; do
  /usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags \
    -c "$root/paper_1604_02153_b200/csrc/$f.cu" -o "$obj/$f.o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
/usr/local/cuda/bin/nvcc $ARCH -shared -o "$out/libvrg_$name.so" "$obj"/*.o -L/usr/local/cuda/lib64 -lcufft -lcudart
echo "built $out/libvrg_$name.so"
