#!/bin/bash
# the round-end driver sequence on one box: GPU tests, smoke, reference arm, device arm
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --impl reference 2>/dev/null | tail -1
timeout 900 python bench.py 2>/dev/null | tail -1
