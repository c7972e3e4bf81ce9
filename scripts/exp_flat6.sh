KVT_FLAT_TRACE=1 python -c "import paper_2605_09490_b200.build as b; b.build(force=True)"
TAG=base timeout 300 python scripts/trace_rt.py
timeout 300 python scripts/trace_slow.py | head -4
python -c "import paper_2605_09490_b200.build as b; b.build(force=True)"
timeout 300 python bench.py --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
