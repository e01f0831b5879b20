# NVMe configs[3]: store alignment 512 vs 4096, queue depth 64 / 128
mkdir -p gpurun_out
for cfg in "512 64" "512 128" "4096 128"; do set -- $cfg
timeout 900 python tools/disk_tier_bench.py 500000 $2 gpurun_out/disk_tier_al$1_qd$2.json $1 > gpurun_out/disk_tier_al$1_qd$2.log 2>&1; echo al$1 qd$2 rc=$?
python -c "import json;r=json.load(open('gpurun_out/disk_tier_al$1_qd$2.json'));print(r['disk_bytes_per_batch']/1e6, r['payload_bytes_per_batch']/1e6, r['serial'], r['pipelined']['queries_per_s'])"
done
