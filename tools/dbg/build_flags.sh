# build the working tree's libstbem.so with extra nvcc flags ($@, e.g. -DSTB_BULK_MINB_D=3) into tools/dbg/alt/
set -e
R=/root/repo
rm -rf $R/tools/dbg/alt; mkdir -p $R/tools/dbg/alt
cd $R/paper_1811_05224_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$R/include "$@" -c assemble.cu -o $R/tools/dbg/alt/assemble.o
cd $R/paper_1811_05224_b200/lib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/dbg/alt/libstbem.so mesh.cpp.o api.cpp.o comm.cu.o $R/tools/dbg/alt/assemble.o linalg.cu.o -ldl -lcudart
rm -f $R/tools/dbg/alt/assemble.o
