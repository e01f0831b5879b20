# small-kernel phase timeline; A/B: all-lane vs one-lane barrier arrives in the MaxSim kernel (C2 bench)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python tools/small_timeline.py 1 > gpurun_out/small_timeline.txt 2>&1; cat gpurun_out/small_timeline.txt
timeout 300 python tools/small_timeline.py 4 >> gpurun_out/small_timeline.txt 2>&1; tail -2 gpurun_out/small_timeline.txt
L=paper_2312_05417_b200/lib/libespn_gpu.so
for v in one all one all; do
  cp tools/ab/libespn_gpu_$v.so $L
  timeout 600 python bench.py --no-cpu-baseline --steps 400 > gpurun_out/bench_n_$v.json 2> gpurun_out/bench_n_$v.err
  python -c "import json;r=json.load(open('gpurun_out/bench_n_$v.json'));print('$v', r['value'],r['e2e']['value'],r['roofline']['frac'],r['roofline']['exclusive']['kernel_ms'],r['clocks']['sm_mhz'],r['clocks']['reasons'])"
done
cp tools/ab/libespn_gpu_all.so $L
