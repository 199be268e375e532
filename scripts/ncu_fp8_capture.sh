#!/usr/bin/env bash
# ncu evidence for the MXFP8 megakernel (fused_moe_kernel<1>): launch list and
# one full capture at the two points VERDICT r1 names (run on the B200 box).
#   bash scripts/ncu_fp8_capture.sh <tag>
set -u
tag=${1:-r2}
out=gpurun_out
mkdir -p "$out"
NCU="ncu --clock-control none"
for pt in "Qwen3-30B-A3B 2048 0.5" "DeepSeek-V3 256 0.5" "Qwen3-30B-A3B 8 0.5"; do
  set -- $pt
  M=$1; S=$2; B=$3
  n="${tag}_fp8_${M%%-*}_s${S}_b${B}"
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file "$out/${n}_launches.csv" python scripts/ncu_point_fp8.py --model "$M" --S "$S" --beta "$B" --reps 3 \
    > "$out/${n}_launches.log" 2>&1
  $NCU --set full --import-source on -k regex:fused_moe -s 2 -c 1 -o "$out/${n}" -f \
    python scripts/ncu_point_fp8.py --model "$M" --S "$S" --beta "$B" --reps 3 > "$out/${n}.log" 2>&1
done
ls -la "$out" | grep "$tag"
