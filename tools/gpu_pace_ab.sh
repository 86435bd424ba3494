mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k persistent > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
run() {
  local label=$1; shift
  echo -n "$label: " >> gpurun_out/ab.log
  env "$@" timeout 300 python bench.py --n $N --steps $K --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
}
N=32768
for K in 300 3000; do
  for pc in 0 74 148 296 592; do run "n$N K$K pace$pc" LTL_PACE=$pc; done
done
run "n$N perlaunch" LTL_NO_PERSIST=1
N=16384
for K in 1000 10000; do
  for pc in 0 148 296; do run "n$N K$K pace$pc" LTL_PACE=$pc; done
done
