#!/bin/bash
# Round-2 evidence: the 7B beta x r grid (every window event-bearing) on the current build,
# and PCIe byte counters of the host-link kernels (stream-mode T1 prefetch, migrate with its offload).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
: > gpurun_out/grid_r02.jsonl
for hbm in 3000 5000 7000; do for ev in 300 500 1000; do
  timeout 300 python bench.py --no-extras --hbm $hbm --evict $ev --steps 192 --warmup 64 2>/dev/null >> gpurun_out/grid_r02.jsonl
done; done
wc -l gpurun_out/grid_r02.jsonl
timeout 900 ncu --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum,dram__bytes_read.sum \
  -k regex:"k_prefetch|k_migrate_rows" -c 12 --csv --log-file gpurun_out/pcie_r02.csv \
  python scripts/prof_step.py --staging 0 --steps 3 > gpurun_out/pcie_r02.log 2>&1; echo "pcie rc=$?"
tail -3 gpurun_out/pcie_r02.log
