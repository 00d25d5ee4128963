#!/bin/bash
timeout 300 python -m pytest tests/test_attention.py -q -x 2>&1 | tail -3
timeout 300 python tools/attn_bench.py 2>&1 | tail -12
