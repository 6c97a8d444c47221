#!/bin/bash
# One GPU evidence pass: parity tests, bench (ours + reference arm), ncu launch
# list of the bench's profile mode, one ncu --set full capture of the top kernels.
# usage (from repo root, on the GPU box): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi_$TAG.txt 2>&1
lscpu > $OUT/lscpu_$TAG.txt 2>&1; nproc >> $OUT/lscpu_$TAG.txt
[ -n "${SKIP_TESTS:-}" ] || { timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_$TAG.log; }
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?" >> $OUT/bench_$TAG.err
[ -n "${SKIP_REF:-}" ] || timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --profile --steps 40 --warmup 3 > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launch exit $?" >> $OUT/ncu_launch_$TAG.log
for k in ${KERNELS:-blend_bwd_kernel blend_fwd_kernel fold_adam_kernel materialize_kernel preprocess_kernel ssim_windows_kernel ssim_pixels_kernel tile_sort_kernel emit_tiles_kernel tile_scan_a_kernel compact_mask_kernel}; do
  SKIP=3; STEPS=2
  [ $k = materialize_kernel ] && { SKIP=0; STEPS=40; }  # (every 32 steps)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $SKIP -c 1 -o $OUT/full_${k}_$TAG -f \
    python bench.py --profile --steps $STEPS --warmup 3 > $OUT/ncu_full_${k}_$TAG.log 2>&1
done
echo done
