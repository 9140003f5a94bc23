#!/bin/bash
# Round-2 ncu evidence (one GPU, each program first run without ncu):
#  1. launch list of one C2 path (gpu__time_duration per launch)
#  2. --set full of the C2 basis GEMMs (the top launches)
#  3. --set full of the fused Gram pass, W = 1 (column pass) and W = 4, 8 (DMMA pass)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
P="python bench.py --path-only --no-cpu-baseline --no-e2e"
if [ -z "$SKIP_LIST" ]; then
timeout 300 $P --steps 1 --warmup 3 > gpurun_out/r02_plain_c2.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches_c2.csv $P --steps 1 --warmup 3 > gpurun_out/r02_ncu_list.log 2>&1
echo "list rc=$?"
fi
if [ -z "$SKIP_GEMM" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma_kernel \
    --launch-skip ${GEMM_SKIP:-100} --launch-count ${GEMM_COUNT:-12} -f -o gpurun_out/r02_gemm_c2 \
    $P --steps 1 --warmup 0 > gpurun_out/r02_ncu_gemm.log 2>&1
echo "gemm rc=$?"
fi
if [ -z "$SKIP_GRAM" ]; then
timeout 300 python tools/gram_pass_bench.py > gpurun_out/r02_gram_plain.txt 2>&1
RP_GRAM_W_ONLY=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"colpass_kernel|gram_dmma_kernel" \
    --launch-skip 3 --launch-count 1 -f -o gpurun_out/r02_gram_w1 \
    python tools/gram_pass_bench.py > gpurun_out/r02_ncu_gram_w1.log 2>&1
RP_GRAM_W_ONLY=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_dmma_kernel" \
    --launch-skip 3 --launch-count 1 -f -o gpurun_out/r02_gram_w8 \
    python tools/gram_pass_bench.py > gpurun_out/r02_ncu_gram_w8.log 2>&1
echo "gram rc=$?"
fi
# Summaries on the box; the reports themselves (tens of MB each) stay behind unless KEEP_REP=1.
for r in r02_gemm_c2 r02_gram_w1 r02_gram_w8; do
  [ -f gpurun_out/$r.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_summary.json 2>/dev/null
  [ -z "$KEEP_REP" ] && rm -f gpurun_out/$r.ncu-rep
done
du -sh gpurun_out
