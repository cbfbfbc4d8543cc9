out=gpurun_out/p2
mkdir -p $out
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
export RB_CODEGEN=2
for cfg in "brown8 6" "katsura6 5" "eco8 4"; do set -- $cfg
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "rb_round_$2/" -k regex:"k_hs_|k_filter" -o $out/$1 python tools/prof_solve.py $1 > $out/ncu_$1.log 2>&1
ncu -i $out/$1.ncu-rep --page raw --csv > $out/$1_raw.csv 2>/dev/null
rm -f $out/$1.ncu-rep
done
ls -la $out
