set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q --timeout=120 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1
