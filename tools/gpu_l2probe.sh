mkdir -p gpurun_out
for n in 8192 10240 12288 16384; do
  echo -n "n$n: " >> gpurun_out/ab.log
  timeout 300 python bench.py --n $n --steps 2000 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
done
LTL_NO_PERSIST=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:ltl_tc_step -s 5 -c 3 --csv --log-file gpurun_out/ncu_8192.csv python bench.py --n 8192 --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
