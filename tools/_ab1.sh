python tools/hs_bench.py katsura6 brown8 eco8 broyden_banded12 --reps 3 2>&1 | grep -v "per round"
for m in 2 3; do echo "== eval minb $m"; RB_CODEGEN_OPTS="-DRB_EVAL_MINB=$m" python tools/hs_bench.py katsura6 brown8 eco8 --reps 3 2>&1 | grep -v "per round"; done
python -m pytest tests/test_full_solves.py tests/test_gpu_parity.py tests/test_gpu_exact.py -m gpu -x -q 2>&1 | tail -2
