#!/usr/bin/env bash
# ncu evidence for profiles/ (run on the B200 box through gpurun; one GPU, one process).
#   bash scripts/ncu_capture.sh <tag>
# Writes gpurun_out/<tag>_*: the per-launch duration list of three sweep
# points and one full capture (details page CSV + .ncu-rep) of the megakernel
# at a decode, an HBM-bound and a tensor-bound point, and of the route kernel.
set -u
tag=${1:-r1}
out=gpurun_out
mkdir -p "$out"
NCU="ncu --clock-control none"
for pt in "1 0.2" "16 1.0" "512 0.2"; do
  set -- $pt
  S=$1; B=$2
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file "$out/${tag}_launches_s${S}_b${B}.csv" python scripts/ncu_point.py --S "$S" --beta "$B" --reps 3 \
    > "$out/${tag}_launches_s${S}_b${B}.log" 2>&1
  $NCU --set full --import-source on -k regex:fused_moe -s 2 -c 1 -o "$out/${tag}_k3_s${S}_b${B}" -f \
    python scripts/ncu_point.py --S "$S" --beta "$B" --reps 3 > "$out/${tag}_k3_s${S}_b${B}.log" 2>&1
  ncu -i "$out/${tag}_k3_s${S}_b${B}.ncu-rep" --page details --csv > "$out/${tag}_k3_s${S}_b${B}_details.csv" 2>/dev/null
done
$NCU --set full --import-source on -k regex:route_kernel -s 2 -c 1 -o "$out/${tag}_route_s512_b0.5" -f \
  python scripts/ncu_point.py --S 512 --beta 0.5 --reps 3 > "$out/${tag}_route.log" 2>&1
ncu -i "$out/${tag}_route_s512_b0.5.ncu-rep" --page details --csv > "$out/${tag}_route_s512_b0.5_details.csv" 2>/dev/null
$NCU --set full --import-source on -k regex:route_kernel -s 2 -c 1 -o "$out/${tag}_route_s1_b0.2" -f \
  python scripts/ncu_point.py --S 1 --beta 0.2 --reps 3 > "$out/${tag}_route1.log" 2>&1
ncu -i "$out/${tag}_route_s1_b0.2.ncu-rep" --page details --csv > "$out/${tag}_route_s1_b0.2_details.csv" 2>/dev/null
ls -la "$out" | grep "$tag"
