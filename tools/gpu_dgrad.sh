#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
A=MGLP_NO_PRESPLIT_DGRAD=1 B=MGLP_NO_PRESPLIT_DGRAD=0 bash tools/gpu_ab_env.sh
CFG=gpt A=MGLP_NO_PRESPLIT_DGRAD=1 B=MGLP_NO_PRESPLIT_DGRAD=0 bash tools/gpu_ab_env.sh
