mkdir -p gpurun_out
timeout 1200 python tools/env_ab.py 4 3 '' 'SPAMM_OZ_SIDE_PRIO=0' 'SPAMM_OZ_SPLIT_CTAS=2' 'SPAMM_OZ_SPLIT_CTAS=1' 'SPAMM_OZ_SIDE_PRIO=0 SPAMM_OZ_SPLIT_CTAS=2' 'SPAMM_OZ_SPLIT_CTAS=0' > gpurun_out/ab.log 2>&1
