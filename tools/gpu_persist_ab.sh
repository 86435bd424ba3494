# persistent sweep vs one launch per generation (GPU box)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for n in 16384 32768; do
  for i in 1 2; do
    for mode in persist perlaunch; do
      env_=""; [[ $mode == perlaunch ]] && env_="LTL_NO_PERSIST=1"
      echo -n "$mode: " >> gpurun_out/ab.log
      env $env_ timeout 300 python bench.py --n $n --steps 500 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
    done
  done
done
