# Balanced-tail tensor-core kernels: parity (selected + split cases), then an A/B of the libraries.
O=gpurun_out/split
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "tc_ or roundtrip or config or determinism or peer or append or balanced" > $O/pytest_sel.log 2>&1; tail -3 $O/pytest_sel.log
VARIANTS="old new new:KVQ_TC_BALANCE=1" NS=1,2,4,8 bash scripts/ab_lib.sh > /dev/null 2>&1
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so
cat gpurun_out/ab/ab.txt
