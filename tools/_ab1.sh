P=paper_1802_00330_b200
python tools/hs_bench.py katsura6 brown8 eco8 --reps 3 2>&1 | grep -v "per round"
for v in u1 u4 m2; do echo "== $v"; RB_LIB_PATH=$P/librootbox_b200_$v.so python tools/hs_bench.py katsura6 brown8 eco8 --reps 3 2>&1 | grep -v "per round"; done
python -m pytest tests/test_full_solves.py tests/test_gpu_parity.py tests/test_gpu_exact.py -m gpu -x -q 2>&1 | tail -2
