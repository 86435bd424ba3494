set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for i in 1 2; do
  for mode in wrap self dist; do
    case $mode in
      wrap) env_="" ; extra="";;
      self) env_="LTL_SELF_RING=1"; extra="";;
      dist) env_=""; extra="--dist";;
    esac
    echo -n "$mode: " >> gpurun_out/ab.log
    env $env_ timeout 300 python bench.py --n 16384 --steps 200 $extra --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
  done
done
