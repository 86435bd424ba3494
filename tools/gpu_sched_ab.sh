# persistent schedules: sweep vs segments vs one launch per generation (GPU box)
mkdir -p gpurun_out
LTL_SEGMENTS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k persistent > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
run() {
  local label=$1; shift
  echo -n "$label: " >> gpurun_out/ab.log
  env "$@" timeout 300 python bench.py --n $N --steps $K --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
}
for n in 16384 32768 65536; do
  N=$n; K=300; [[ $n == 65536 ]] && K=60
  for i in 1 2; do
    run "n$n sweep16" X=1
    run "n$n segments" LTL_SEGMENTS=1
    run "n$n perlaunch" LTL_NO_PERSIST=1
  done
done
