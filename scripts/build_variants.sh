# build compile-time variants of the library into scripts/so_var/lib_<name>.so (A/B timing via TM_LIB_PATH)
#   bash scripts/build_variants.sh name1 "DEFS1" name2 "DEFS2" ...
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  args=""; for d in $defs; do args="$args -D$d"; done
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared \
    $args -I include -o scripts/so_var/lib_$name.so paper_2508_15601_b200/csrc/api.cu > scripts/so_var/$name.log 2>&1 &
done
wait
ls -la scripts/so_var/*.so
