mkdir -p gpurun_out
for i in 1 2; do
  for n in 24576 32768; do
    for m in default force; do
      env_=X=1; [[ $m == force ]] && env_=LTL_FORCE_PERSIST=1
      echo -n "$m n$n: " >> gpurun_out/ab.log
      env $env_ timeout 300 python bench.py --n $n --steps 300 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
    done
  done
done
