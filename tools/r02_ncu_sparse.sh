#!/bin/bash
# ncu --set full of the sparse Gram passes (C4 CSR, 128 right-hand columns), summarized on the box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/sparse_ncu.py 1.0 128 > gpurun_out/sparse_plain.txt 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none -k regex:"pass1_kernel|pass2_kernel" --launch-skip 80 --launch-count 4 -f \
    -o gpurun_out/r02_sparse python tools/sparse_ncu.py 1.0 128 > gpurun_out/r02_ncu_sparse.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_sparse.ncu-rep > gpurun_out/r02_sparse_summary.json 2>/dev/null
rm -f gpurun_out/r02_sparse.ncu-rep
python - <<'P'
import json
for r in json.load(open("gpurun_out/r02_sparse_summary.json")):
    print(r["kernel"][:40], r.get("gpu__time_duration.sum"), "dram r/w", r.get("dram__bytes_read.sum"), r.get("dram__bytes_write.sum"),
          "L2 hit", r.get("lts__t_sector_hit_rate.pct"))
P
