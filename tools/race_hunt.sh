#!/bin/bash
# Concurrency hunt (GPU box): which set-up product is wrong under stream
# priorities, and does it survive disabling device-memory reuse (no free /
# same-stream-only pool reuse), TMA, PDL or lazy loading.  (compute-sanitizer
# is closed on this pool: runs under it have left GPUs needing a reset.)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/race_hunt${HUNT_TAG}.txt
: > $out
run() { echo "== $*" >> $out; timeout 300 env "$@" >> $out 2>&1; echo "rc=$?" >> $out; }
if [ -n "$HUNT_CASES" ]; then
  eval "$HUNT_CASES"
else
run python tools/race_hunt.py 3 stream_priorities=1
run RP_LEAK_ALLOC=1 python tools/race_hunt.py 2 stream_priorities=1
run RP_LEAK_ALLOC=2 python tools/race_hunt.py 3 stream_priorities=1
run RP_POOL_STRICT=1 python tools/race_hunt.py 3 stream_priorities=1
run CUDA_MODULE_LOADING=EAGER python tools/race_hunt.py 2 stream_priorities=1
run RP_GEMM_TMA=0 python tools/race_hunt.py 2 stream_priorities=1
run RP_GEMM_PDL=0 python tools/race_hunt.py 2 stream_priorities=1
run python tools/race_hunt.py 2 stream_priorities=1,gram_overlap_tma=0
run python tools/race_hunt.py 2 default
run tools/tma_race_bin 4 8
fi
