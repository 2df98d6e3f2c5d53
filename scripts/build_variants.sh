# Build alternative libfmm2d.so variants of near.cu for tuning (loaded with FMM2D_LIB=...).
set -e
ARCH="-gencode arch=compute_100a,code=sm_100a"
for v in "$@"; do
  name=$(echo "$v" | tr -c 'A-Za-z0-9_\n' '_' )
  mkdir -p build/var_$name
  nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden $v \
       -c paper_1006_2269_b200/csrc/near.cu -o build/var_$name/near.o
  nvcc $ARCH -shared -o build/var_$name/libfmm2d.so build/api.o build/expansions.o build/lists.o build/tree.o build/var_$name/near.o
  echo "build/var_$name/libfmm2d.so"
done
