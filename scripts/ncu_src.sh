#!/usr/bin/env bash
# Source-level (CUDA line) ncu capture of one forced megakernel config:
#   bash scripts/ncu_src.sh <tag> <one.py args...>
set -u
tag=$1; shift
out=gpurun_out
ncu --set full --import-source on --clock-control none -k regex:fused_moe -s 2 -c 1 -o "$out/$tag" -f \
  python scripts/one.py "$@" > "$out/$tag.log" 2>&1
ncu -i "$out/$tag.ncu-rep" --page source --csv --print-source cuda > "$out/${tag}_cuda.csv" 2>/dev/null
ncu -i "$out/$tag.ncu-rep" --page raw --csv > "$out/${tag}_raw.csv" 2>/dev/null
ncu -i "$out/$tag.ncu-rep" --page details --csv > "$out/${tag}_details.csv" 2>/dev/null
