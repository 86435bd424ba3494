mkdir -p gpurun_out
for i in 1 2 3; do
  for v in A B; do
    echo -n "$v: " >> gpurun_out/ab.log
    LTL_LIB=build/ab/$v.so timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
  done
  echo -n "B dist: " >> gpurun_out/ab.log
  LTL_LIB=build/ab/B.so timeout 300 python bench.py --dist --steps 1000 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
done
