#!/bin/bash
# Build A/B variants of libssm_b200.so (same sources, different kernel macros)
# into paper_1306_3277_b200/lib/variants/<name>/ -- measured with
# profiles/run_variants.sh under gpurun (SSM_LIB_PATH selects the build).
set -e
cd "$(dirname "$0")/.."
ARCH="-gencode arch=compute_100a,code=sm_100a"
build() {  # name, extra nvcc flags
  local name=$1; shift
  local out=paper_1306_3277_b200/lib/variants/$name
  mkdir -p $out/obj
  for f in paper_1306_3277_b200/csrc/*.cu; do
    nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $f -o $out/obj/$(basename $f .cu).o &
  done
  wait
  nvcc $ARCH -shared -o $out/libssm_b200.so $out/obj/*.o -lcudart -lnvrtc
  rm -rf $out/obj
  echo built $name
}
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  [ "$name" = "$flags" ] && flags=""
  build $name $flags
done
