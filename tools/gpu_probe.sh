mkdir -p gpurun_out
SPAMM_HTRACE=1 timeout 300 python tools/ncu_solve.py 4 > gpurun_out/htrace.log 2>&1
