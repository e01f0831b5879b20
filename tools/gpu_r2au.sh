# new default (no pad-patch warp, 16 warps): full suite, smoke, bench, sanitizers
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_au.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_au.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_au.json 2> gpurun_out/bench_au.err; echo bench=$?
python -c "import json;r=json.load(open('gpurun_out/bench_au.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive']['frac'],r['gather_hbm_gbs'],r['clocks'],r['gpu_launches'])"
for i in 1 2; do timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
SAN_TIMEOUT=900 bash tools/sanitize.sh
