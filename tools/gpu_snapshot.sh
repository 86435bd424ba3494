mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_snapshot.py -x -q > gpurun_out/pytest_snap.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_snap.log
df -h /dev/shm /tmp > gpurun_out/df.txt 2>&1
timeout 900 python tools/snapshot_bench.py --n 16384 32768 --dir /dev/shm > gpurun_out/snapshot_shm.json 2> gpurun_out/snapshot.err
timeout 900 python tools/snapshot_bench.py --n 16384 --dir /tmp > gpurun_out/snapshot_tmp.json 2>> gpurun_out/snapshot.err
