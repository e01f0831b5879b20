# final code: full GPU suite, smoke, default bench, reference arm, sanitizers
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_ah.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_ah.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ah.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_ah.log
timeout 600 python bench.py > gpurun_out/bench_ah.json 2> gpurun_out/bench_ah.err; echo bench=$?
python -c "import json;r=json.load(open('gpurun_out/bench_ah.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive']['frac'],r['gather_hbm_gbs'],r['clocks'],r['gpu_launches'])"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ah_ref.json 2> gpurun_out/bench_ah_ref.err; echo ref=$?
SAN_TIMEOUT=900 bash tools/sanitize.sh
