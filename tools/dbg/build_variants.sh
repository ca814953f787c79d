# build one libstbem.so per flag set into tools/dbg/alt_<i>/ (A/B runs of assemble.cu variants):
#   bash tools/dbg/build_variants.sh "-DX=1" "-DX=1 -DY=2" ...
set -e
R=/root/repo
i=0
for flags in "$@"; do
  d=$R/tools/dbg/alt_$i; rm -rf $d; mkdir -p $d; echo "$flags" > $d/flags.txt
  ( cd $R/paper_1811_05224_b200/csrc &&
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr -I$R/include $flags -c assemble.cu -o $d/assemble.o &&
    cd $R/paper_1811_05224_b200/lib &&
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libstbem.so \
      mesh.cpp.o api.cpp.o comm.cu.o $d/assemble.o linalg.cu.o -ldl -lcudart && rm -f $d/assemble.o ) &
  i=$((i+1))
done
wait
