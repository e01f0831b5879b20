# A/B: issuing lanes per bulk-copy producer warp (ESPN_PLANES 2 / 4 = production / 8 / 32)
mkdir -p gpurun_out
VARIANTS="prod planes2 planes8 planes32" bash tools/gpu_r2be.sh
