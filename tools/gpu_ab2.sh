# correctness with the worktree library, then interleaved A/B (build/ab/A.so, B.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for n in 16384 32768; do
  for i in 1 2; do
    for v in A B; do
      echo -n "n$n $v: " >> gpurun_out/ab.log
      LTL_LIB=build/ab/$v.so timeout 300 python bench.py --n $n --steps 300 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
    done
  done
done
