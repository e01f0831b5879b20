# adopt 128-doc units at d=32: full GPU suite, smoke, bench (C2 + C1), sanitizers
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_u128.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_u128.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_u128_c2.json 2> gpurun_out/bench_u128_c2.err; echo bench=$?; cat gpurun_out/bench_u128_c2.json
bash tools/sanitize.sh
