mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for i in 1 2; do
  for v in A B; do
    echo -n "$v dist: " >> gpurun_out/ab.log
    LTL_LIB=build/ab/$v.so timeout 300 python bench.py --dist --steps 1000 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
  done
  echo -n "B single: " >> gpurun_out/ab.log
  LTL_LIB=build/ab/B.so timeout 300 python bench.py --steps 1000 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
done
