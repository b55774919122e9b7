# build a variant library: tools/build_variant.sh NAME "-DFOO=1 ..." -> abtest/NAME/librama_b200.so
set -e
NAME=$1; shift
D=abtest/$NAME; mkdir -p $D/obj
for f in paper_2109_01838_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
    --expt-relaxed-constexpr $@ -c $f -o $D/obj/$b.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/librama_b200.so $D/obj/*.o -lcudart
echo $D/librama_b200.so
