run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=$1 tools/dist_check.py $2 $3 2>&1 | grep -A2 'init\|run 3:\|re-upload\|more'; }
echo "== init check, gens 3 (the failing sequence)"; DIFF=1 run 29681 1024 1024
echo "== download rank 0"; DIFF=1 SKIP_INIT_CHECK=1 DOWNLOAD_ONLY=0 run 29682 4096 4096
