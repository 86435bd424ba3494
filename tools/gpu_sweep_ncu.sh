# DRAM bytes / L2 hit rate: persistent sweep vs per-launch at 32768^2 (GPU box)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum
for u in 16 32; do
  LTL_SWEEP_UNITS=$u timeout 600 ncu --metrics $M --clock-control none -k regex:ltl_tc_step --csv \
    --log-file gpurun_out/ncu_sweep$u.csv python bench.py --n 32768 --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
LTL_NO_PERSIST=1 timeout 600 ncu --metrics $M --clock-control none -k regex:ltl_tc_step -c 6 --csv \
  --log-file gpurun_out/ncu_perlaunch.csv python bench.py --n 32768 --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for u in 8 4; do
  echo -n "n32768 P$u: " >> gpurun_out/ab.log
  LTL_SWEEP_UNITS=$u timeout 300 python bench.py --n 32768 --steps 300 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
  echo -n "n16384 P$u: " >> gpurun_out/ab.log
  LTL_SWEEP_UNITS=$u timeout 300 python bench.py --n 16384 --steps 300 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
done
