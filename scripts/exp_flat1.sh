python -c "import __graft_entry__ as g; g.build()"
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read()); L=d['L14']; print(sys.argv[1], 'loop', round(L['loop_done'][1]-L['first_stage'][1],2), 'epi', L['epilogue_us_per_cta'], 'cta_o', L['epi_to_cta_o_us'], 'deltas', d['layer_end_deltas_us'][10:14])" "$1"; }
timeout 300 python scripts/trace_flat.py | summ base
KVTIER_NOPDL=1 timeout 300 python scripts/trace_flat.py | summ nopdl
KVTIER_SPIN=20000 timeout 300 python scripts/trace_flat.py | summ spin20k
KVTIER_SPIN=1000 timeout 300 python scripts/trace_flat.py | summ spin1k
