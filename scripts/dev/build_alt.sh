# Dev tool: an A/B variant of libpbg.so with extra nvcc defines, for PBG_LIB comparisons.
#   bash scripts/dev/build_alt.sh NAME -DFOO   -> paper_1410_2788_b200/_lib/alt_NAME/libpbg.so
set -e
NAME=$1; shift
R=$(cd "$(dirname "$0")/../.." && pwd)
O=$R/paper_1410_2788_b200/_lib/alt_$NAME
mkdir -p $O
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -I$R/include -I$R/paper_1410_2788_b200/csrc "$@" -c $R/paper_1410_2788_b200/csrc/sweep.cu -o $O/sweep.o
objs="$O/sweep.o"
for f in slab schemes_extra capi assemble vacuum; do objs="$objs $R/paper_1410_2788_b200/_lib/obj/$f.o"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o $O/libpbg.so -lcufft
echo $O/libpbg.so
