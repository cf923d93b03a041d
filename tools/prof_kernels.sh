#!/bin/bash
# ncu --set full captures of the first N kernels matching a regex per case
# (GPU box, one GPU):  tools/prof_kernels.sh <outdir> "name|regex|count|env|profile_op args" ...
# Keeps the raw-page CSV (and the source page of the first kernel), removes
# the .ncu-rep (gpurun_out/ is pulled back only below 64 MiB).
out=$1; shift
mkdir -p "$out"
for c in "$@"; do
  IFS='|' read -r name rx cnt envs args <<< "$c"
  env $envs timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s 3 -c "$cnt" \
    -o "/tmp/$name" -f python tools/profile_op.py $args > "$out/$name.log" 2>&1
  ncu -i "/tmp/$name.ncu-rep" --page raw --csv > "$out/${name}_raw.csv" 2>/dev/null
  rm -f "/tmp/$name.ncu-rep"
done
