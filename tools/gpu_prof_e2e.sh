timeout 300 python tools/e2e_prof.py broyden_tri6 > gpurun_out/e2e_prof.log 2>&1; echo e2e=$?
RB_TRACE=1 timeout 300 python tools/trace_run.py broyden_tri6 > gpurun_out/trace_bt6.log 2>&1; echo trace=$?
