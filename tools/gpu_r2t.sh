# full GPU suite (small-kernel fuzz, C++ disk tier), smoke, final default bench + reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_t.log 2>&1; echo pytest=$?; tail -8 gpurun_out/pytest_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_t.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke_t.log
timeout 600 python bench.py > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err; echo bench=$?
python -c "import json;r=json.load(open('gpurun_out/bench_t.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive']['frac'],r['gather_hbm_gbs'],r['clocks'],r['gpu_launches'])"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_t_ref.json 2> gpurun_out/bench_t_ref.err; echo ref=$?; head -c 300 gpurun_out/bench_t_ref.json
