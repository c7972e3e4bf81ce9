KVT_FLAT_TRACE=1 python -c "import paper_2605_09490_b200.build as b; b.build(force=True)"
TAG=base timeout 300 python scripts/trace_rt.py
TAG=if1 KVTIER_INFLIGHT=1 timeout 300 python scripts/trace_rt.py
