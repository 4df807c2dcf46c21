#!/bin/bash
# gpu_round.sh, then summarise on the box (ncu reports are too large to bring back):
# profiles/<dest> + profiles/ncu_traffic.json are copied into gpurun_out/<dest>_profiles/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-round}
DEST=${2:-r01_$TAG}
bash scripts/gpu_round.sh "$TAG"
python scripts/save_profile.py "$TAG" "$DEST" > gpurun_out/save_profile_$TAG.log 2>&1
for t in c64 g xy; do
  [ -f gpurun_out/prof_${t}_$TAG.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/prof_${t}_$TAG.ncu-rep > profiles/$DEST/ncu_${t}_summary.txt
done
for f in bench_c64 configs smoke; do :; done
cp gpurun_out/bench_c64_$TAG.log profiles/$DEST/bench_c64.json 2>/dev/null
cp gpurun_out/configs_$TAG.jsonl profiles/$DEST/configs.jsonl 2>/dev/null
cp gpurun_out/smoke_$TAG.log profiles/$DEST/smoke.txt 2>/dev/null
cp gpurun_out/xy_$TAG.log profiles/$DEST/xy.jsonl 2>/dev/null
cp gpurun_out/latency_$TAG.log profiles/$DEST/latency.txt 2>/dev/null
cp gpurun_out/bench_mp2_$TAG.log profiles/$DEST/bench_mp2_one_device.log 2>/dev/null
mkdir -p gpurun_out/${DEST}_profiles
cp -r profiles/$DEST/. gpurun_out/${DEST}_profiles/
cp profiles/ncu_traffic.json gpurun_out/${DEST}_profiles/ncu_traffic.json
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
