# A/B: mbarrier wait flavour (ESPN_WAIT_MODE: 0 try_wait no hint, 1 try_wait 10 ms hint = production, 2 test_wait spin)
mkdir -p gpurun_out
VARIANTS="prod wait0 wait2" bash tools/gpu_r2be.sh
