# sweep chunk size / flag cost (GPU box); libraries from tools/ab_build.sh
mkdir -p gpurun_out
run() {  # label env... -- bench args
  local label=$1; shift
  echo -n "$label: " >> gpurun_out/ab.log
  env "$@" timeout 300 python bench.py --n $N --steps 300 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
}
for n in 32768 16384; do
  N=$n
  run "n$n P32" LTL_LIB=build/ab/P.so
  run "n$n P16" LTL_LIB=build/ab/P.so LTL_SWEEP_UNITS=16
  run "n$n P64" LTL_LIB=build/ab/P.so LTL_SWEEP_UNITS=64
  run "n$n P128" LTL_LIB=build/ab/P.so LTL_SWEEP_UNITS=128
  run "n$n P256" LTL_LIB=build/ab/P.so LTL_SWEEP_UNITS=256
  run "n$n NF32" LTL_LIB=build/ab/NF.so
  run "n$n NF128" LTL_LIB=build/ab/NF.so LTL_SWEEP_UNITS=128
  run "n$n perlaunch" LTL_LIB=build/ab/P.so LTL_NO_PERSIST=1
done
