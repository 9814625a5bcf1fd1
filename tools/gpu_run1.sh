set -x
nvidia-smi; free -g; nproc; lscpu | grep -E "Model name|Socket|Core|Thread"
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -40
for v in 0 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --variant $v; done
