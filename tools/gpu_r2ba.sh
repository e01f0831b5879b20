# A/B unit size with round-balanced sizing: served step + bench (value, exclusive launch, p50)
mkdir -p gpurun_out
L=paper_2312_05417_b200/lib/libespn_gpu.so
for v in cur u96 u64 cur u96 u64; do cp tools/ab/libespn_gpu_$v.so $L; printf "%s " $v; timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
for v in cur u96 u64 cur u96 u64; do
  cp tools/ab/libespn_gpu_$v.so $L
  timeout 600 python bench.py --no-cpu-baseline --steps 300 > gpurun_out/bench_ab_$v.json 2> gpurun_out/bench_ab_$v.err
  python -c "import json;r=json.load(open('gpurun_out/bench_ab_$v.json'));print('$v', round(r['value']),round(r['e2e']['value']),round(r['roofline']['frac'],4),r['roofline']['exclusive']['kernel_ms'],round(r['p50_batch_ms'],4),r['clocks']['sm_mhz'],r['clocks']['reasons'])"
done
cp tools/ab/libespn_gpu_cur.so $L
