#!/bin/bash
# Per-generation time of the recursion's P product (fused update epilogue) for every candidate tile, C2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/pg
for t in auto 1 2 3 4 6 11 13 14 15 16 17; do
  if [ $t = auto ]; then unset RP_PGEMM_TILE; else export RP_PGEMM_TILE=$t; fi
  RP_GEMM_LOG=gpurun_out/pg/log_$t.txt timeout 300 python bench.py --config c2 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e \
     --dump-gemm gpurun_out/pg/prof_$t.json > gpurun_out/pg/bench_$t.json 2> gpurun_out/pg/err_$t.txt
  python tools/gemm_per_launch.py gpurun_out/pg/prof_$t.json gpurun_out/pg/log_$t.txt > gpurun_out/pg/tbl_$t.txt 2>&1
  echo "tile $t: $(tail -n 1 gpurun_out/pg/tbl_$t.txt)"
done
python - <<'P'
import glob, re
rows = {}
for f in sorted(glob.glob("gpurun_out/pg/tbl_*.txt")):
    t = f.split("_")[-1][:-4]
    for ln in open(f):
        p = ln.split()
        if len(p) == 11 and p[6] == "2":
            rows.setdefault(int(p[1]), {})[t] = float(p[7])
tiles = ["auto", "1", "2", "3", "4", "6", "11", "13", "14", "15", "16", "17"]
print("   N " + " ".join(f"{t:>6s}" for t in tiles) + "   best")
for n in sorted(rows):
    r = rows[n]
    best = min((v, t) for t, v in r.items() if t != "auto")
    print(f"{n:4d} " + " ".join(f"{r.get(t, float('nan')):6.1f}" for t in tiles) + f"   {best[1]} ({best[0]:.1f})")
P
