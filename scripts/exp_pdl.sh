python scripts/sweep_attn.py --splits 8 --variants 4,0 > gpurun_out/exp_default.log 2>&1
python scripts/sweep_attn.py --splits 8 --variants 4,0 --env KVTIER_PDL_PRE=1 > gpurun_out/exp_pre1.log 2>&1
python scripts/sweep_attn.py --splits 8 --variants 4,0 --env KVTIER_PDL_PRE=0 > gpurun_out/exp_pre0.log 2>&1
python scripts/sweep_attn.py --splits 8 --variants 4,0 --env KVTIER_NOPDL=1 > gpurun_out/exp_nopdl.log 2>&1
KVTIER_PDL_PRE=1 python scripts/trace_attn.py --split 8 --variant 4 > gpurun_out/trace12.log 2>&1
KVTIER_NOPDL=1 python scripts/trace_attn.py --split 8 --variant 4 >> gpurun_out/trace12.log 2>&1
