set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo EXIT $? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_ozaki -s 40 -c 1 -o gpurun_out/k4z python tools/ncu_solve.py 4 > gpurun_out/ncu_k4z.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_ozaki32 -s 40 -c 1 -o gpurun_out/k4z32 python tools/ncu_solve.py 3 > gpurun_out/ncu_k4z32.log 2>&1
ls -la gpurun_out
