# 96-doc units at d=32 (NU 3) + round-balanced unit sizing: GPU suite, smoke, bench, sanitizers, ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_u96.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_u96.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
for i in 1 2 3; do timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
timeout 600 python bench.py > gpurun_out/bench_r2_v8_c2.json 2> gpurun_out/bench_r2_v8_c2.err; echo bench=$?
python -c "import json;r=json.load(open('gpurun_out/bench_r2_v8_c2.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive']['kernel_ms'],r['p50_batch_ms'],r['clocks'],r['check'])"
timeout 600 python bench.py --impl reference > gpurun_out/bench_r2_v8_c2_reference_arm.json 2> gpurun_out/ref.err; echo ref=$?
timeout 600 python bench.py --config c1 > gpurun_out/bench_r2_v8_c1.json 2> gpurun_out/c1.err; echo c1=$?
python -c "import json;r=json.load(open('gpurun_out/bench_r2_v8_c1.json'));print('c1',r['value'],r['e2e']['value'],r.get('p50_batch_ms'),r['config'].get('kernel'))"
bash tools/sanitize.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 5 -c 1 -o gpurun_out/prof_maxsim_u96 -f python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_full_u96.log 2>&1; echo ncufull=$?
ncu -i gpurun_out/prof_maxsim_u96.ncu-rep --page raw --csv > gpurun_out/maxsim_raw_u96.csv 2>&1; echo raw=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|plan|finalize|wait|gather" -c 120 --csv --log-file gpurun_out/launches_u96.csv python bench.py --steps 20 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_launch_u96.log 2>&1; echo ncu=$?
