# build libstbem.so from the sources of revision $1 into tools/dbg/alt/ (A/B runs against the tree)
set -e
R=/root/repo; REV=$1
rm -rf $R/tools/dbg/alt; mkdir -p $R/tools/dbg/alt/src
git -C $R archive $REV paper_1811_05224_b200/csrc include | tar -x -C $R/tools/dbg/alt/src
cd $R/tools/dbg/alt/src/paper_1811_05224_b200/csrc
objs=""
for s in mesh.cpp api.cpp comm.cu assemble.cu linalg.cu; do
  [ -f $s ] || continue
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$R/tools/dbg/alt/src/include -c $s -o $s.o &
  objs="$objs $s.o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/dbg/alt/libstbem.so $objs -ldl -lcudart
rm -rf $R/tools/dbg/alt/src
