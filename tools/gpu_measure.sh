#!/bin/bash
# Round measurement bundle (run under gpurun from the repo root): parity suite, the
# bench line (ours + reference arm), the bench launch list and ncu --set full captures
# of the dominant kernels of the headline and the large BASELINE configs.
set -u
out=gpurun_out/m
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt
python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
python bench.py --steps 200 --warmup 10 > $out/bench.json 2> $out/bench.err
python bench.py --impl reference --steps 20 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $out/ncu_bench.log 2>&1
export RB_CODEGEN=2
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "rb_round_3/" -o $out/bt6_r3 \
    python tools/prof_solve.py broyden_tri6 > $out/ncu_bt6.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "rb_round_5/" -o $out/k6_r5 \
    python tools/prof_solve.py katsura6 > $out/ncu_k6.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "rb_round_6/" -o $out/brown8_r6 \
    python tools/prof_solve.py brown8 > $out/ncu_brown8.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "rb_round_4/" --nvtx-include "rb_round_5/" \
    -o $out/eco8_r4r5 python tools/prof_solve.py eco8 > $out/ncu_eco8.log 2>&1
ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "rb_round_2/" -o $out/banded12_r2 \
    python tools/prof_solve.py broyden_banded12 > $out/ncu_banded12.log 2>&1
# raw metrics + per-line source counters as CSV; the reports themselves stay on the box
for r in bt6_r3 k6_r5 brown8_r6 eco8_r4r5 banded12_r2; do
    if [ -f $out/$r.ncu-rep ]; then
        ncu -i $out/$r.ncu-rep --page raw --csv > $out/${r}_raw.csv 2>/dev/null
        ncu -i $out/$r.ncu-rep --page details --csv > $out/${r}_details.csv 2>/dev/null
        rm -f $out/$r.ncu-rep
    fi
done
du -sh $out; ls -la $out
