for i in 1 2; do
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('base value %.2f' % d['value'])"
QGS_OVERLAP_FWD=1 timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('overlap value %.2f' % d['value'])" || tail -5 /tmp/b.log
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo --no-cpu > /tmp/d.log 2>&1; echo "dist rc=$?"; tail -1 /tmp/d.log | cut -c1-400
