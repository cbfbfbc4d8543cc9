# Round-end measurement bundle (dev tool): bench line, reference arm, launch list and
# ncu --set full captures exported to CSV (reports deleted: gpurun_out/ is capped at 64 MiB).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref2.log 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-other-configs --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
cap() {  # name config rounds
  RB_GRAPH=0 timeout 900 ncu --set full --nvtx --nvtx-include "rb_round_$3/" --clock-control none --import-source on -f -o /tmp/$1 python tools/prof_run.py $2 $3 > gpurun_out/ncu_$1.log 2>&1; echo ncu_$1=$?
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$1.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/ncu_details_$1.csv 2>/dev/null
  rm -f /tmp/$1.ncu-rep
}
cap bt6_r3 broyden_tri6 3
cap k6_r5 katsura6 5
cap eco8_r5 eco8 5
