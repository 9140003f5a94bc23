#!/bin/bash
# Round-2 concurrency probes on one B200 (binaries prebuilt into tools/probe_bin by nvcc here).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B=tools/probe_bin
R=${REPS:-48}
{
echo "## tma_check (pipeline verifier, no GEMM): two streams, low/high priority"
timeout 300 $B/tma_check 60 1 8 | tail -n 12
echo "## tma_check: two streams, one priority"
timeout 300 $B/tma_check 30 0 8 | tail -n 6
echo "## tma_check: two processes time-sharing the GPU, one priority each"
( timeout 300 $B/tma_check 40 0 8 | tail -n 6 | sed 's/^/[p1] /' ) &
( timeout 300 $B/tma_check 40 0 8 | tail -n 6 | sed 's/^/[p2] /' ) &
wait
for v in base fence order gmap; do
  echo "## tma_race mode 4 (path SYRK beside 40 TMA GEMMs), side low / chain high priority: variant $v"
  timeout 600 $B/race_$v 4 $R 1 | grep -v "mismatches 0, chain mismatches 0" | tail -n 12
done
echo "## tma_race mode 4, one priority, variant base"
timeout 600 $B/race_base 4 $R 0 | grep -v "mismatches 0, chain mismatches 0" | tail -n 6
echo "## tma_race mode 4: two processes, one priority each, variant base"
( timeout 600 $B/race_base 4 24 0 | grep -v "mismatches 0, chain mismatches 0" | tail -n 6 | sed 's/^/[p1] /' ) &
( timeout 600 $B/race_base 4 24 0 | grep -v "mismatches 0, chain mismatches 0" | tail -n 6 | sed 's/^/[p2] /' ) &
wait
} > gpurun_out/tma_probe.txt 2>&1
cat gpurun_out/tma_probe.txt
