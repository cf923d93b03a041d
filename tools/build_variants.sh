#!/bin/bash
# Build tuning variants of libsk200 (Helmholtz kernels only):
#   tools/build_variants.sh eb16_nt1_mb0 eb8_nt2_mb1 ...
# -> paper_2604_04644_b200/libsk200_<name>.so, used by tools/tune_eb.py.
set -e
cd "$(dirname "$0")/../paper_2604_04644_b200/csrc"
for v in "$@"; do
  eb=$(echo "$v" | sed -E 's/eb([0-9]+)_nt([0-9]+)_mb([0-9]+)/\1/')
  nt=$(echo "$v" | sed -E 's/eb([0-9]+)_nt([0-9]+)_mb([0-9]+)/\2/')
  mb=$(echo "$v" | sed -E 's/eb([0-9]+)_nt([0-9]+)_mb([0-9]+)/\3/')
  make -j"$(nproc)" BUILD=/tmp/sk200_build_$v LIB=../libsk200_$v.so LINEINFO= \
    EXTRA="-DSK_ONLY_HELM -DSK_EB_FIXED=$eb -DSK_NT_DIV=$nt -DSK_MINB=$mb" > /dev/null 2>&1
  echo "built libsk200_$v.so"
done
