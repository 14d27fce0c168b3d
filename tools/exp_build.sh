# Build an experimental variant of the library into tools/exp/<name>.so
# (used with WLCS_LIB_PATH=...); extra nvcc flags after the name.
set -e
name=$1; shift
mkdir -p tools/exp/obj_$name
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC $*"
for f in paper_1306_4627_b200/csrc/*.cu; do b=$(basename $f .cu); $NV -c $f -o tools/exp/obj_$name/$b.o & done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/exp/$name.so tools/exp/obj_$name/*.o build/obj/facade_*.cpp.o -lpthread -ldl -lrt
rm -rf tools/exp/obj_$name
