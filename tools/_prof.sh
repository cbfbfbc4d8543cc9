out=gpurun_out/p
mkdir -p $out
export RB_CODEGEN=2
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "rb_round_6/" -k regex:"k_hs_lin_tps|k_hs_sweep|k_hs_eval" -o $out/b8 python tools/prof_solve.py brown8 > $out/ncu.log 2>&1
ncu -i $out/b8.ncu-rep --page raw --csv > $out/b8_raw.csv 2>/dev/null
for k in k_hs_lin_tps k_hs_sweep k_hs_eval; do
  ncu -i $out/b8.ncu-rep -k regex:$k --page source --print-source cuda,sass --csv > $out/b8_${k}_src.csv 2>/dev/null
done
rm -f $out/b8.ncu-rep
ls -la $out
