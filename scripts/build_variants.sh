# Build alternative libfmm2d.so variants for tuning (loaded with FMM2D_LIB=...).
# usage: build_variants.sh <source-stem> "<defines>" ["<defines>" ...]
set -e
ARCH="-gencode arch=compute_100a,code=sm_100a"
stem=$1; shift
for v in "$@"; do
  name=$(echo "$stem $v" | tr -c 'A-Za-z0-9_\n' '_' )
  mkdir -p build/var_$name
  nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden $v \
       -c paper_1006_2269_b200/csrc/$stem.cu -o build/var_$name/$stem.o
  objs=""
  for o in api expansions lists near rr shard tree; do
    if [ "$o" = "$stem" ]; then objs="$objs build/var_$name/$stem.o"; else objs="$objs build/$o.o"; fi
  done
  nvcc $ARCH -shared -o build/var_$name/libfmm2d.so $objs
  echo "build/var_$name/libfmm2d.so"
done
