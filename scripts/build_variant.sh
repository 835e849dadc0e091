# Build ab/libkvq_<name>.so: attn_tc.cu recompiled with extra flags, linked with the in-tree objects of the
# other sources (run `python -m paper_2601_04719_b200.build` first).  Experiments only.
#   bash scripts/build_variant.sh NAME "-DFLAG ..."
set -e
N=$1; F=$2
mkdir -p ab/obj_$N
NCCL_INC=$(python -c "import sysconfig,os;print(os.path.join(sysconfig.get_paths()['purelib'],'nvidia','nccl','include'))")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true \
  -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr $F -I include -I $NCCL_INC \
  -c paper_2601_04719_b200/csrc/attn_tc.cu -o ab/obj_$N/attn_tc.o
objs=$(ls paper_2601_04719_b200/build/*.o | grep -v attn_tc.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/libkvq_$N.so $objs ab/obj_$N/attn_tc.o -ldl -lpthread
echo ab/libkvq_$N.so
