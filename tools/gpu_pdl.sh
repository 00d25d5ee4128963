#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
A=MGLP_NO_PDL=1 B=MGLP_NO_PDL=0 bash tools/gpu_ab_env.sh
CFG=mt A=MGLP_NO_PDL=1 B=MGLP_NO_PDL=0 bash tools/gpu_ab_env.sh
