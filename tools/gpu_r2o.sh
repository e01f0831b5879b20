# small kernel v3 (two warps per doc, L2 dedup hash, smem two-level merge); suite; sanitizers
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests/test_small_gpu.py -x -q > gpurun_out/pytest_o_small.log 2>&1; echo small=$?; tail -5 gpurun_out/pytest_o_small.log
timeout 300 python tools/small_timeline.py 1 > gpurun_out/small_timeline_o.txt 2>&1; timeout 300 python tools/small_timeline.py 4 >> gpurun_out/small_timeline_o.txt 2>&1; cat gpurun_out/small_timeline_o.txt
for k in 1 3; do timeout 120 ./tools/c1_latency $k; done > gpurun_out/c1_latency_o.txt 2>&1; cat gpurun_out/c1_latency_o.txt
timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 200 --warmup 10 > gpurun_out/bench_o_c1.json 2> gpurun_out/bench_o_c1.err; echo c1=$?
python -c "import json;r=json.load(open('gpurun_out/bench_o_c1.json'));print(r['value'],r['e2e']['value'],r['p50_batch_ms'],r['roofline']['kernel_ms'],r['roofline']['exclusive']['kernel_ms'],r['config']['kernel'])"
compute-sanitizer --tool racecheck ./tools/racecheck_probe > gpurun_out/racecheck_probe_o.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_o.log 2>&1; echo pytest=$?; tail -8 gpurun_out/pytest_o.log
SAN_TIMEOUT=900 bash tools/sanitize.sh
