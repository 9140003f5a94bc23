#!/bin/bash
# A/B of the set-up overlap (Gram SYRK beside sketch + Cholesky chain) once concurrent TMA grids are exact.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{
echo "## option A/B, C2 (tools/option_ab.py, 10 reps, 2 rounds)"
timeout 1200 python tools/option_ab.py c2 10 default "stream_priorities=1" "gram_overlap_occ=1" \
  "gram_overlap_occ=1,gram_overlap_tile=1" "gram_overlap_occ=1,gram_overlap_tile=1,stream_priorities=1" \
  "gram_overlap_occ=2,gram_overlap_tile=3,stream_priorities=1" \
  "gram_overlap_occ=1,gram_overlap_tile=1,gram_overlap_split=16,stream_priorities=1" \
  "gram_after_sketch=1,stream_priorities=1" "gram_after_sketch=1,gram_overlap_occ=1,gram_overlap_tile=1,stream_priorities=1" \
  "gram_overlap_split=16,stream_priorities=1" 2>&1 | tail -n 22
echo "## stress: bitwise vs the serialized run"
timeout 900 python tools/race_stress.py c2 30 "stream_priorities=1" "gram_overlap_occ=1,gram_overlap_tile=1,stream_priorities=1" 2>&1 | tail -n 3
echo "## per-launch GEMM table (recursion), C2"
RP_GEMM_LOG=gpurun_out/gemm.log timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --dump-gemm gpurun_out/gemm_prof.json > gpurun_out/bench_c2_tbl.json 2> gpurun_out/bench_c2_tbl.err
python tools/gemm_per_launch.py gpurun_out/gemm_prof.json gpurun_out/gemm.log
} > gpurun_out/overlap_ab.txt 2>&1
tail -n 200 gpurun_out/overlap_ab.txt
