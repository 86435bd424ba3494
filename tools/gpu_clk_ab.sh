mkdir -p gpurun_out
run() {
  local label=$1; shift
  echo -n "$label: " >> gpurun_out/ab.log
  env "$@" timeout 300 python bench.py --n $N --steps $K --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
}
N=32768; K=3000
run "sweep" X=1
run "segments" LTL_SEGMENTS=1
run "perlaunch" LTL_NO_PERSIST=1
N=16384; K=10000
run "sweep" X=1
run "perlaunch" LTL_NO_PERSIST=1
