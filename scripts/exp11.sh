#!/bin/bash
T=${1:-c13}
KVT_TRACE_LOOP=1 python -c "from paper_2605_09490_b200 import build; build.build(force=True)" > gpurun_out/build_${T}_tl.log 2>&1
timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace_${T}_tl.log 2>&1
timeout 300 python scripts/trace_attn.py --split 8 --variant 4 > gpurun_out/trace_${T}_tl_v4.log 2>&1
