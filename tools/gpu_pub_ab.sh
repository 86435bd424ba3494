# cost of the persistent kernel's flag waits / publication (GPU box)
mkdir -p gpurun_out
run() {
  local label=$1; shift
  echo -n "$label: " >> gpurun_out/ab.log
  env "$@" timeout 300 python bench.py --n $N --steps $K --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
}
N=32768; K=300
for i in 1 2; do
  for v in P NF NFP; do
    run "sweep $v" LTL_LIB=build/ab/$v.so
    run "segments $v" LTL_LIB=build/ab/$v.so LTL_SEGMENTS=1
  done
  run "perlaunch" LTL_LIB=build/ab/P.so LTL_NO_PERSIST=1
done
