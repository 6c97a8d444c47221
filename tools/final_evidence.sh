set -u
KERNELS="blend_bwd_kernel blend_fwd_kernel adam_kernel adam_rot_kernel fold_visible_kernel preprocess_kernel ssim_windows_kernel ssim_pixels_kernel" bash tools/gpu_round.sh r01f
python tools/cfg5_sweep.py --out gpurun_out/cfg5_sweep_r01f.json > gpurun_out/cfg5f.log 2>&1
python tools/consensus_bench.py --config cfg3 --out gpurun_out/consensus_cfg3_r01f.json > gpurun_out/cons3f.log 2>&1
python tools/consensus_bench.py --config cfg4 --out gpurun_out/consensus_cfg4_r01f.json > gpurun_out/cons4f.log 2>&1
timeout 1500 python tools/cfg1_parity.py --out gpurun_out/cfg1_parity_r01f.json > gpurun_out/cfg1f.log 2>&1
echo all-done
