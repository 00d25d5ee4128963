nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -25
timeout 600 python bench.py --config tiny --steps 5 --warmup 3 2>&1 | tail -3
timeout 900 python bench.py --config bert --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
