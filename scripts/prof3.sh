ncu --set full --clock-control none --import-source on -k regex:k_decode_merge -s 30 -c 1 -o gpurun_out/merge_full python scripts/prof_step.py --split 8 --variant 0 > gpurun_out/p3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 30 -c 1 -o gpurun_out/attn_v5 python scripts/prof_step.py --split 8 --variant 0 > gpurun_out/p4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv python scripts/prof_step.py --split 8 --variant 0 --steps 3 > /dev/null 2>&1
