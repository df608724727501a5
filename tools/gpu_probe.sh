mkdir -p gpurun_out
SPAMM_TF_PROF=1 timeout 300 python tools/ncu_solve.py 4 > gpurun_out/tf_prof.log 2>&1
SPAMM_CULL_PROF=1 timeout 300 python tools/ncu_solve.py 4 > gpurun_out/cull_prof.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo EXIT $? >> gpurun_out/pytest_gpu.log
timeout 1200 python tools/env_ab.py 4 3 'SPAMM_LIB_PATH=ab/libspamm_head.so' '' > gpurun_out/ab.log 2>&1
timeout 300 python tools/critical_path.py 4 > gpurun_out/critical_path.log 2>&1
