set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for qp in auto rounded; do
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --query-precision $qp > gpurun_out/bench_$qp.json 2> gpurun_out/bench_$qp.err; echo bench_$qp=$?
done
