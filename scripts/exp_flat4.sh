python -c "import __graft_entry__ as g; g.build()"
summ() { python -c "
import json,sys; d=json.loads(sys.stdin.read()); L=d['L14']; dl=d['layer_end_deltas_us']
print(sys.argv[1], 'first', round(L['first_stage'][1]-L['pdl_wait'][1],2), 'loop', round(L['loop_done'][1]-L['first_stage'][1],2), 'loopmax', round(L['loop_done'][2]-L['first_stage'][1],2), 'side_score', round(L['side_score_done'][1]-L['pdl_wait'][1],2), 'layer_mean', round(sum(dl[4:])/len(dl[4:]),2))" "$1"; }
for fv in 0 1 2; do KVTIER_FVAR=$fv timeout 300 python scripts/trace_flat.py | summ fvar$fv; done
KVTIER_L2PF_MB=0 timeout 300 python scripts/trace_flat.py | summ nopf
timeout 300 python bench.py --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
