mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
LTL_NO_PERSIST=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ltl_tc_step -s 3 -c 1 \
    -o gpurun_out/prof_pk -f python bench.py --n 16384 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pk.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_pk.log
