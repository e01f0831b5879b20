# small kernel v4 (fp32 quad staging + paired fp32 ops): parity, C1 bench, latency, timeline
timeout 900 python -m pytest tests/test_small_gpu.py tests/test_fuzz_gpu.py tests/test_sharded_gpu.py -q -x > gpurun_out/pytest_ao.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_ao.log
timeout 300 python bench.py --no-cpu-baseline --config c1 --steps 200 --warmup 10 > gpurun_out/bench_ao_c1.json 2> gpurun_out/bench_ao_c1.err; echo c1=$?
python -c "import json;r=json.load(open('gpurun_out/bench_ao_c1.json'));print(r['value'],r['e2e']['value'],r['p50_batch_ms'],r['roofline']['kernel_ms'],r['roofline']['exclusive']['kernel_ms'],r['clocks']['sm_mhz'])"
for k in 3 1; do timeout 120 ./tools/c1_latency $k; done
timeout 300 python tools/small_timeline.py 1 2>&1 | tail -2
