# ptxas register / spill report of one csrc file (default attn_tc.cu), extra nvcc flags from $EXTRA.
F=${1:-attn_tc.cu}
R=/root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ftz=false -prec-div=true -prec-sqrt=true \
  -Xcompiler -fPIC --expt-relaxed-constexpr $EXTRA -I $R/include \
  -I $(python -c "import sysconfig,os;print(os.path.join(sysconfig.get_paths()['purelib'],'nvidia','nccl','include'))") \
  -Xptxas -v -c $R/paper_2601_04719_b200/csrc/$F -o /tmp/ptxas_check.o 2>&1 | grep -E "Compiling entry|spill|Used" | paste - - - | sed 's/ptxas info    ://g' | cut -c1-250
