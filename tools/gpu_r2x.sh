# pipelined loader: parity subset, role profile, server timing, default bench
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_server_gpu.py tests/test_fuzz_gpu.py -x -q > gpurun_out/pytest_x.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_x.log
timeout 300 python tools/role_profile.py on 2>&1 | tail -18
for i in 1 2; do timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err; echo bench=$?
python -c "import json;r=json.load(open('gpurun_out/bench_x.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive'],r['clocks'])"
