#!/bin/bash
# ncu --set full captures of selected launches (name regex, skip count) for one step at 2^LG
LG=${1:-28}; TAG=${2:-r01}; shift 2
mkdir -p gpurun_out
while [ $# -gt 1 ]; do
  K=$1; S=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}\$" -s $S -c 1 \
      -o gpurun_out/${TAG}_${K}_s${S} python tools/prof_step.py $LG 1 > gpurun_out/${TAG}_${K}_s${S}.log 2>&1
done
ls gpurun_out | grep $TAG
