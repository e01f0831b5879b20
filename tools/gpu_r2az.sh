# round-balanced unit sizing with 128-doc units at d=32: GPU suite, smoke, served step, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_u128b.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_u128b.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
for i in 1 2; do timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
timeout 600 python bench.py > gpurun_out/bench_u128b_c2.json 2> gpurun_out/bench_u128b_c2.err; echo bench=$?
python -c "import json;r=json.load(open('gpurun_out/bench_u128b_c2.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive']['kernel_ms'],r['p50_batch_ms'],r['clocks']['sm_mhz'],r['clocks']['reasons'])"
