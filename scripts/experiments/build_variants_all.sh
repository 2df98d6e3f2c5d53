# Build whole-library variants (every .cu compiled with the given defines) into build/var_*/libfmm2d.so
# usage: build_variants_all.sh "<defines>" ["<defines>" ...]
set -e
ARCH="-gencode arch=compute_100a,code=sm_100a"
for v in "$@"; do
  name=$(echo "all $v" | tr -c 'A-Za-z0-9_\n' '_' )
  mkdir -p build/var_$name
  objs=""
  for o in api expansions lists near rr shard tree; do
    nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden $v \
         -c paper_1006_2269_b200/csrc/$o.cu -o build/var_$name/$o.o &
    objs="$objs build/var_$name/$o.o"
  done
  wait
  nvcc $ARCH -shared -o build/var_$name/libfmm2d.so $objs
  echo "build/var_$name/libfmm2d.so"
done
