# build an alternative libstbem.so from the committed (HEAD) moments.cuh into tools/dbg/alt/ (A/B runs)
set -e
R=/root/repo
rm -rf $R/tools/dbg/alt; mkdir -p $R/tools/dbg/alt/x/csrc $R/tools/dbg/alt/include; cp $R/include/stbem.h $R/tools/dbg/alt/include/
git -C $R show HEAD:paper_1811_05224_b200/csrc/moments.cuh > $R/tools/dbg/alt/x/csrc/moments.cuh
for f in internal.h special.cuh special_coeffs.h moment_coeffs.h potential.cuh initial.cuh assemble.cu; do cp $R/paper_1811_05224_b200/csrc/$f $R/tools/dbg/alt/x/csrc/; done
cd $R/tools/dbg/alt/x/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$R/include -c assemble.cu -o $R/tools/dbg/alt/assemble.o
cd $R/paper_1811_05224_b200/lib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/dbg/alt/libstbem.so mesh.cpp.o api.cpp.o comm.cu.o $R/tools/dbg/alt/assemble.o linalg.cu.o -ldl -lcudart
rm -rf $R/tools/dbg/alt/x $R/tools/dbg/alt/include $R/tools/dbg/alt/assemble.o
