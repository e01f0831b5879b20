# A/B: d=32 work-unit size (UNITMAX 64 / 96 / 128+NU2): parity then served C2 step
mkdir -p gpurun_out
L=paper_2312_05417_b200/lib/libespn_gpu.so
for v in u96 u128; do
  cp tools/ab/libespn_gpu_$v.so $L
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py tests/test_server_gpu.py -x -q -m gpu > gpurun_out/par_$v.log 2>&1; echo "$v parity=$? $(tail -1 gpurun_out/par_$v.log)"
done
for v in cur u96 u128 cur u96 u128 cur u96 u128; do cp tools/ab/libespn_gpu_$v.so $L; printf "%s " $v; timeout 300 python tools/server_knobs.py 0 on 2>&1 | tail -1; done
for v in cur u96 u128; do
  cp tools/ab/libespn_gpu_$v.so $L
  timeout 600 python bench.py --no-cpu-baseline --steps 400 > gpurun_out/bench_u_$v.json 2> gpurun_out/bench_u_$v.err
  python -c "import json;r=json.load(open('gpurun_out/bench_u_$v.json'));print('$v', r['value'],r['e2e']['value'],r['roofline']['frac'],r['clocks']['sm_mhz'],r['clocks']['reasons'])"
done
cp tools/ab/libespn_gpu_cur.so $L
