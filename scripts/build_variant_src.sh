# Build ab/libkvq_<name>.so with one source file recompiled with extra flags (experiments only):
#   bash scripts/build_variant_src.sh NAME SRC.cu "-DFLAG ..."
set -e
N=$1; SRC=$2; F=$3
mkdir -p ab/obj_$N
NCCL_INC=$(python -c "import sysconfig,os;print(os.path.join(sysconfig.get_paths()['purelib'],'nvidia','nccl','include'))")
O=ab/obj_$N/${SRC%.cu}.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true \
  -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr $F -I include -I $NCCL_INC -c paper_2601_04719_b200/csrc/$SRC -o $O
objs=$(ls paper_2601_04719_b200/build/*.o | grep -v "/${SRC%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/libkvq_$N.so $objs $O -ldl -lpthread
echo ab/libkvq_$N.so
