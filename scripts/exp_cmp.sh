python -c "import paper_2605_09490_b200.build as b; b.build(force=True)"
b() { timeout 300 python bench.py --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step']*1000/28,2), 'us/layer', round(d['roofline']['frac'],3))"; }
KVTIER_FLAT=1 b flat
KVTIER_FLAT=1 KVTIER_NOSCORE=1 b flat_noscore
KVTIER_FLAT=0 b split
KVTIER_FLAT=0 KVTIER_NOSCORE=1 b split_noscore
KVTIER_FLAT=1 KVTIER_INFLIGHT=1 b flat_if1
