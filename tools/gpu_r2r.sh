# disk tier tests + NVMe configs[3] benchmark (queue depth 64 and 16)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_disk_tier_gpu.py -x -q > gpurun_out/pytest_r_disk.log 2>&1; echo disk=$?; tail -3 gpurun_out/pytest_r_disk.log
timeout 900 python tools/disk_tier_bench.py 500000 64 gpurun_out/disk_tier_qd64.json > gpurun_out/disk_tier_qd64.log 2>&1; echo disk64=$?; tail -3 gpurun_out/disk_tier_qd64.log
timeout 900 python tools/disk_tier_bench.py 500000 16 gpurun_out/disk_tier_qd16.json > gpurun_out/disk_tier_qd16.log 2>&1; echo disk16=$?; tail -2 gpurun_out/disk_tier_qd16.log
