# final verification of the round's last tree: GPU suite, smoke, C2 bench + reference arm, C2 launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_final.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_r2_v11_c2.json 2> gpurun_out/bench_r2_v11_c2.err; echo bench=$?
python -c "import json;r=json.load(open('gpurun_out/bench_r2_v11_c2.json'));print(r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive']['frac'],r['p50_batch_ms'],r['clocks'],r['check'])"
timeout 600 python bench.py --impl reference > gpurun_out/bench_r2_v11_c2_reference_arm.json 2> gpurun_out/ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"maxsim|plan|finalize|wait|gather" -c 120 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 20 --warmup 3 --preroll-s 0 --no-cpu-baseline --server off > gpurun_out/ncu_launch_final.log 2>&1; echo ncu=$?
