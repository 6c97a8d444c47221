# Full evidence pass on the GPU box: tests, bench (+ reference arm), ncu launch
# list and full captures (tools/gpu_round.sh), the other BASELINE configs'
# drivers and the kernel timeline. usage: bash tools/final_evidence.sh [tag]
set -u
TAG=${1:-r02e}
bash tools/gpu_round.sh $TAG
timeout 900 python tools/timeline.py --out gpurun_out/timeline_$TAG.json > gpurun_out/timeline_$TAG.log 2>&1
timeout 900 python tools/timeline.py --e2e --out gpurun_out/timeline_e2e_$TAG.json > gpurun_out/timeline_e2e_$TAG.log 2>&1
timeout 1200 python tools/cfg5_sweep.py --out gpurun_out/cfg5_sweep_$TAG.json > gpurun_out/cfg5_$TAG.log 2>&1
timeout 900 python tools/consensus_bench.py --config cfg3 --out gpurun_out/consensus_cfg3_$TAG.json > gpurun_out/cons3_$TAG.log 2>&1
timeout 1200 python tools/consensus_bench.py --config cfg4 --out gpurun_out/consensus_cfg4_$TAG.json > gpurun_out/cons4_$TAG.log 2>&1
for c in cfg2 cfg3 cfg4; do
  timeout 1500 python tools/blocks_bench.py --config $c --blocks 1,2,4,8 --out gpurun_out/blocks_${c}_$TAG.json > gpurun_out/blocks_${c}_$TAG.log 2>&1
done
timeout 1500 python tools/cfg1_parity.py --out gpurun_out/cfg1_parity_$TAG.json > gpurun_out/cfg1_$TAG.log 2>&1
echo all-done
