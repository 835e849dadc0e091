# Tail-cutting variants: parity of the tensor-core paths (incl. forced cuts), then an A/B of the libraries.
O=gpurun_out/split
mkdir -p $O
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so
timeout 900 python -m pytest tests -m gpu -x -q -k "tc_ or roundtrip or config or determinism or peer or balanced or plain_launches" > $O/pytest_sel.log 2>&1; tail -3 $O/pytest_sel.log
VARIANTS="old new" NS=1,2,4,8 bash scripts/ab_lib.sh > /dev/null 2>&1
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so
grep -v metrics gpurun_out/ab/ab.txt
