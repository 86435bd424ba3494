#!/bin/bash
# After the prologue fix: u8 vs 4-bit cells on one box, bench lines of both.
set -u
mkdir -p gpurun_out
for i in 1 2; do timeout 300 python tools/pk_time.py 32768 cat cat-4bit; timeout 300 python tools/pk_time.py 16384 cat cat-4bit; done
for e in cat cat-4bit; do
  timeout 900 python bench.py --engine $e --steps 20 --warmup 5 > gpurun_out/bench_c2_$e.json 2> gpurun_out/bench_c2_$e.err; echo "bench $e rc=$?"
  python tools/bench_line.py < gpurun_out/bench_c2_$e.json
  python -c "import json; d=json.loads(open('gpurun_out/bench_c2_$e.json').read().splitlines()[-1]); print('e2e %.3e'%d['e2e']['value'], 'cpu', d.get('cpu_baseline',{}).get('value'))"
done
