# DRAM bytes per generation of long persistent launches vs per-launch (GPU box)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
for mode in sweep segments; do
  env $([[ $mode == segments ]] && echo LTL_SEGMENTS=1 || echo X=1) timeout 900 ncu --metrics $M --clock-control none -k regex:ltl_tc_step --csv \
    --log-file gpurun_out/ncu_drift_$mode.csv python bench.py --n 32768 --steps 100 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
LTL_NO_PERSIST=1 timeout 900 ncu --metrics $M --clock-control none -k regex:ltl_tc_step -c 8 --csv \
  --log-file gpurun_out/ncu_drift_perlaunch.csv python bench.py --n 32768 --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
