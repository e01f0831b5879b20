# non-served launches capped at 64-doc units: GPU suite, served step, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_cap.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_cap.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
for i in 1 2; do timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; timeout 300 python tools/server_knobs.py 0 off 2>&1 | tail -1; done
timeout 600 python bench.py > gpurun_out/bench_r2_v9_c2.json 2> gpurun_out/bench_r2_v9_c2.err; echo bench=$?
python -c "import json;r=json.load(open('gpurun_out/bench_r2_v9_c2.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive']['kernel_ms'],r['roofline']['exclusive']['frac'],r['p50_batch_ms'],r['clocks'],r['check'])"
timeout 600 python bench.py --server off --no-cpu-baseline > gpurun_out/bench_r2_v9_c2_noserver.json 2>/dev/null; python -c "import json;r=json.load(open('gpurun_out/bench_r2_v9_c2_noserver.json'));print('noserver',r['value'],r['e2e']['value'],r['p50_batch_ms'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc -s 5 -c 1 -o gpurun_out/prof_maxsim_cap -f python bench.py --steps 10 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_full_cap.log 2>&1; echo ncufull=$?
ncu -i gpurun_out/prof_maxsim_cap.ncu-rep --page raw --csv > gpurun_out/maxsim_raw_cap.csv 2>&1; echo raw=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|plan|finalize|wait|gather" -c 120 --csv --log-file gpurun_out/launches_cap.csv python bench.py --steps 20 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_launch_cap.log 2>&1; echo ncu=$?
