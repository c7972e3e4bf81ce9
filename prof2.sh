ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 30 -c 1 -o gpurun_out/attn_s8v2 python scripts/prof_step.py --split 8 --variant 2 > gpurun_out/p1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 30 -c 1 -o gpurun_out/attn_s1v2 python scripts/prof_step.py --split 1 --variant 2 > gpurun_out/p2.log 2>&1
