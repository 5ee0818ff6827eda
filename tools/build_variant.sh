# Build a librig variant with extra nvcc defines into variants/$1.so (performance experiments).
# usage: bash tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
mkdir -p variants/obj_$1
for f in paper_1710_07769_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden $2 -c $f -o variants/obj_$1/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$1.so variants/obj_$1/*.o -Xcompiler -fPIC -lcudart
