#!/bin/bash
# Final round-2 measurement batch (one B200): bench lines of every config, the reference arm, ncu evidence.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python bench.py --config c2 --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err; echo "c1 rc=$?"
timeout 1200 python bench.py --config c3 --steps 3 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 1500 python bench.py --config c4 --steps 2 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --impl reference --config c2 --steps 2 --warmup 1 > $O/bench_reference_c2.json 2> $O/bench_reference_c2.err; echo "ref rc=$?"
for c in c1 c2 c3 c4 c5; do python - <<P
import json
try:
    j=json.load(open("$O/bench_$c.json"))
    print("$c", round(j["value"],5), "e2e", round(j["e2e"]["value"],5), "frac", round(j["roofline"]["frac"],3), "cpu", round(j["cpu_baseline"]["value"],1), j["cpu_baseline"]["cores"], "launches", j["gpu_launches"], j["clocks"])
except Exception as e:
    print("$c failed", e)
P
done
