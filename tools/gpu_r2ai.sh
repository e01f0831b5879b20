# N>1 harness check on a 1-GPU box (ranks share GPU 0; not a performance number): spawn, rendezvous,
# max-over-ranks timing, sharded exchange over gloo, replica placement
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ai_c2_g2.json 2> gpurun_out/bench_ai_c2_g2.err; echo c2g2=$?; head -c 1200 gpurun_out/bench_ai_c2_g2.json; echo; tail -3 gpurun_out/bench_ai_c2_g2.err
timeout 900 python bench.py --gpus 2 --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ai_c3_g2.json 2> gpurun_out/bench_ai_c3_g2.err; echo c3g2=$?; head -c 1500 gpurun_out/bench_ai_c3_g2.json; echo; tail -3 gpurun_out/bench_ai_c3_g2.err
