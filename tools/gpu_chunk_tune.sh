mkdir -p gpurun_out
for i in 1 2; do
  for u in 12 16 20 24; do
    echo -n "units $u: " >> gpurun_out/ab.log
    LTL_SWEEP_UNITS=$u timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
  done
done
