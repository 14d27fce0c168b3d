# Build the library of git revision REV into tools/exp/NAME.so (for A/B runs
# with WLCS_LIB_PATH).  Usage: exp_build_rev.sh REV NAME
set -e
rev=$1; name=$2; repo=$(pwd); wt=/tmp/wt_$name
rm -rf $wt; git worktree prune
git worktree add -q --detach $wt $rev
cd $wt
python3 paper_1306_4627_b200/csrc/gen_rowstep.py > paper_1306_4627_b200/csrc/rowstep.cuh
mkdir -p obj
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Iinclude -Xcompiler -fPIC"
for f in paper_1306_4627_b200/csrc/*.cu; do b=$(basename $f .cu); $NV -c $f -o obj/$b.o & done
for f in paper_1306_4627_b200/csrc/*.cpp; do b=$(basename $f .cpp); g++ -std=c++20 -O2 -fPIC -Iinclude -c $f -o obj/$b.cpp.o & done
wait
mkdir -p $repo/tools/exp
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $repo/tools/exp/$name.so obj/*.o -lpthread -ldl -lrt
cd $repo; git worktree remove --force $wt
