export RB_CODEGEN=sync RB_CODEGEN_LINEINFO=1 RB_GRAPH=0
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "rb_round_3/" -k regex:k_hs_fused --clock-control none -f -o /tmp/hsf python tools/prof_run.py broyden_tri6 6 > gpurun_out/ncu_hsf.log 2>&1
ncu -i /tmp/hsf.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_hsf_source.csv 2>/dev/null
ncu -i /tmp/hsf.ncu-rep --page raw --csv > gpurun_out/ncu_hsf_raw.csv 2>/dev/null
ls -la gpurun_out/ncu_hsf*
