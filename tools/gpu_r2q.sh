# full GPU suite; disk-tier (NVMe) configs[3] benchmark
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -8 gpurun_out/pytest_q.log
df -hT /tmp | tail -1; free -g | head -2; nproc
timeout 900 python tools/disk_tier_bench.py 500000 64 gpurun_out/disk_tier_qd64.json > gpurun_out/disk_tier_qd64.log 2>&1; echo disk64=$?; tail -3 gpurun_out/disk_tier_qd64.log
