#!/bin/bash
# Confirmation of the stage-release fix (fence.proxy.async before the "empty" arrive).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B=tools/probe_bin
{
for v in fixed nofence; do
  echo "## tma_race mode 4, side low / chain high priority: $v"
  timeout 900 $B/race_$v 4 ${REPS:-128} 1 | grep -v "mismatches 0, chain mismatches 0" | tail -n 8
done
echo "## tma_race mode 0 (both TMA, default layouts), priorities: fixed"
timeout 900 $B/race_fixed 0 64 1 | grep -v "mismatches 0, chain mismatches 0" | tail -n 4
echo "## two processes time-sharing, one priority each: fixed"
( timeout 900 $B/race_fixed 4 64 0 | grep -v "mismatches 0, chain mismatches 0" | tail -n 4 | sed 's/^/[p1] /' ) &
( timeout 900 $B/race_fixed 4 64 0 | grep -v "mismatches 0, chain mismatches 0" | tail -n 4 | sed 's/^/[p2] /' ) &
wait
echo "## two processes time-sharing, one priority each: nofence"
( timeout 900 $B/race_nofence 4 64 0 | grep -v "mismatches 0, chain mismatches 0" | tail -n 4 | sed 's/^/[p1] /' ) &
( timeout 900 $B/race_nofence 4 64 0 | grep -v "mismatches 0, chain mismatches 0" | tail -n 4 | sed 's/^/[p2] /' ) &
wait
echo "## C2 path stress, every x(lambda) bitwise vs the serialized run (tools/race_stress.py)"
RP_FACTOR_CHAIN_TMA=1 timeout 900 python tools/race_stress.py c2 40 "gram_overlap_tma=1" "gram_overlap_tma=1,gram_after_sketch=1" default 2>&1 | tail -n 6
echo "## C2 option A/B (tools/option_ab.py)"
timeout 600 python tools/option_ab.py c2 10 default "gram_overlap_tma=1" 2>&1 | tail -n 4
echo "## same with the factor chain on the TMA kernel"
RP_FACTOR_CHAIN_TMA=1 timeout 600 python tools/option_ab.py c2 10 default "gram_overlap_tma=1" "gram_overlap_tma=1,gram_after_sketch=1" 2>&1 | tail -n 6
echo "## fused Gram pass (tools/gram_pass_bench.py)"
timeout 600 python tools/gram_pass_bench.py 2>&1 | tail -n 14
} > gpurun_out/tma_probe2.txt 2>&1
cat gpurun_out/tma_probe2.txt
