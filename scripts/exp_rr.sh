python -c "import __graft_entry__ as g; g.build()"
b() { timeout 300 python bench.py --no-extras $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step']*1000/28,2), 'us/layer', round(d['value']))"; }
KVTIER_RR=2 b rr2
KVTIER_RR=1 b rr1
KVTIER_RR=2 b rr2_s9 "--split 9"
KVTIER_RR=2 b rr2_s6 "--split 6"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
