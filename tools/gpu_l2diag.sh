mkdir -p gpurun_out
for i in 1 2; do
for v in N L2; do
  for n in 16384 32768; do
    echo -n "$v n$n: " >> gpurun_out/ab.log
    LTL_LIB=build/ab/$v.so timeout 300 python bench.py --n $n --steps 300 --no-cpu-baseline 2>>gpurun_out/ab.err | python tools/bench_line.py >> gpurun_out/ab.log
  done
done
done
LTL_LIB=build/ab/L2.so LTL_NO_PERSIST=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:ltl_tc_step -s 5 -c 2 --csv --log-file gpurun_out/ncu_l2.csv python bench.py --n 32768 --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
