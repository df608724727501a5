# GPU suite + cfg4 bench (+ optional extra command in $EXTRA)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo EXIT $? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/critical_path.py 4 > gpurun_out/critical_path.log 2>&1
