mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for i in 1 2 3; do
  for v in A B; do
    for n in 16384 32768; do
      echo -n "$v n$n: " >> gpurun_out/ab.log
      LTL_LIB=build/ab/$v.so timeout 300 python bench.py --n $n --steps 500 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
    done
  done
done
