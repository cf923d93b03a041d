#!/bin/bash
# Build tuning variants of libsk200 restricted to one operator class:
#   tools/build_variants.sh op0_eb8_nt1_mb1_cap4 op1_eb16_nt2_mb1_cap8_rd9 ...
# keys: op (SK_ONLY_OP: 0 Helmholtz/stiffness, 1 mass, 2 bwd_trans only,
# 4 phys_deriv, 6 non-collocated Helmholtz), eb (tile elements), nt (thread
# divisor), mb (min-blocks rule on/off), cap (CTAs/SM cap), rd (ragged
# dispatch max order), lowreg (low-register metric sweep), mtma / htma /
# htmar (TMA pipelines: mass, deformed / regular Helmholtz), mwg / mwc /
# mwb (warp-tile mass), eo (even-odd from order), td (tet slice dispatch),
# s (row stride), iu (items unroll), ps (persistent), ring, ch, pf, ...
# (see the case list below); omitted keys keep the sk_tune.h tables.
# -> paper_2604_04644_b200/libsk200_<name>.so, used by tools/tune_eb.py.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
# build from a snapshot of the sources, so editing them meanwhile is safe
SNAP=$(mktemp -d /tmp/sk200_src_XXXX)
mkdir -p "$SNAP/paper_2604_04644_b200" && cp -r "$ROOT/include" "$SNAP/" && cp -r "$ROOT/paper_2604_04644_b200/csrc" "$SNAP/paper_2604_04644_b200/"
rm -rf "$SNAP/paper_2604_04644_b200/csrc/build"
cd "$SNAP/paper_2604_04644_b200/csrc"
for v in "$@"; do
  extra=""
  for kv in ${v//_/ }; do
    k=$(echo "$kv" | sed -E 's/^([a-z]+)[0-9]+$/\1/')
    n=$(echo "$kv" | sed -E 's/^[a-z]+([0-9]+)$/\1/')
    case $k in
      op) extra="$extra -DSK_ONLY_OP=$n" ;;
      eb) extra="$extra -DSK_EB_FIXED=$n" ;;
      nt) extra="$extra -DSK_NT_DIV=$n" ;;
      mb) extra="$extra -DSK_MINB=$n" ;;
      cap) extra="$extra -DSK_MINB_CAP=$n" ;;
      rd) extra="$extra -DSK_RAGGED_MAXP=$n" ;;
      pd) extra="$extra -DSK_GEO_PD=$n" ;;
      ps) extra="$extra -DSK_PERSIST=$n" ;;
      eo) extra="$extra -DSK_EO_MINP=$n" ;;
      ch) extra="$extra -DSK_GEO_CH=$n" ;;
      td) extra="$extra -DSK_TET_DISPATCH_MAXP=$n" ;;
      sl) extra="$extra -DSK_STREAM_LD=$n" ;;
      s) extra="$extra -DSK_S2=$n" ;;
      pf) extra="$extra -DSK_GEO_PF=$n" ;;
      sp) extra="$extra -DSK_SPLIT_MINP=$n" ;;
      iu) extra="$extra -DSK_ITEMS_UNROLL=$n" ;;
      wp) extra="$extra -DSK_PRISM_WP=$n" ;;
      smt) extra="$extra -DSK_SMT=$n" ;;
      rrl) extra="$extra -DSK_RRL=$n" ;;
      ring) extra="$extra -DSK_GEO_RING=$n" ;;
      dminb) extra="$extra -DSK_DENSE_MINB=$n" ;;
      dpf) extra="$extra -DSK_DENSE_PF=$n" ;;
      lowreg) extra="$extra -DSK_M2_LOWREG=$n" ;;
      mwg) extra="$extra -DSK_MASS_WARP_G=$n" ;;
      mwc) extra="$extra -DSK_MASS_WARP_WPC=$n" ;;
      mwb) extra="$extra -DSK_MASS_WARP_MINB=$n" ;;
      mtma) extra="$extra -DSK_MASS_TMA=$n" ;;
      htma) extra="$extra -DSK_HELM_TMA=$n" ;;
      htmar) extra="$extra -DSK_HELM_TMA_REG=$n" ;;
    esac
  done
  make -j"$(nproc)" BUILD=/tmp/sk200_build_$v LIB=$ROOT/paper_2604_04644_b200/libsk200_$v.so LINEINFO= EXTRA="$extra" > /tmp/sk200_build_$v.log 2>&1 \
    && echo "built libsk200_$v.so ($extra)" || { echo "FAILED $v"; tail -5 /tmp/sk200_build_$v.log; }
done
