# disk tier (ESPN_TABLE_DISK_TIER + espn_gpu_prefetch_rows) tests; full suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_disk_tier_gpu.py -x -q > gpurun_out/pytest_p_disk.log 2>&1; echo disk=$?; tail -30 gpurun_out/pytest_p_disk.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_p.log 2>&1; echo pytest=$?; tail -8 gpurun_out/pytest_p.log
