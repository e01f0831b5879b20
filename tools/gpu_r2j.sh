# round-2 re-entry (container re-created): full GPU suite, smoke, default bench, reference arm, sanitizers
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_j.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_j.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_j.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke_j.log
timeout 600 python bench.py > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err; echo bench=$?
tail -3 gpurun_out/bench_j.err; cat gpurun_out/bench_j.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_j_ref.json 2> gpurun_out/bench_j_ref.err; echo ref=$?; cat gpurun_out/bench_j_ref.json
SAN_TIMEOUT=700 bash tools/sanitize.sh
