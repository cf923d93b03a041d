#!/bin/bash
# ncu --set full captures of one k_tile launch per case (GPU box):
#   tools/prof_batch.sh <outdir> "op shape P E" ...
out=$1; shift
mkdir -p "$out"
for c in "$@"; do
  set -- $c
  name="${1}_${2}${3}"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 2 -c 1 \
    -o "$out/$name" -f python tools/profile_op.py --op $1 --shape $2 --order $3 --elements $4 --reps 3 \
    > "$out/$name.log" 2>&1
  ncu -i "$out/$name.ncu-rep" --page raw --csv > "$out/${name}_raw.csv" 2>/dev/null
done
