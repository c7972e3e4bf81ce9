KVT_FLAT_TRACE=1 python -c "import paper_2605_09490_b200.build as b; b.build(force=True)"
for cfg in "0 0" "0 1" "0 2" "3 1" "3 2" "3 3"; do set -- $cfg
  TAG="fvar$1_if$2" KVTIER_FVAR=$1 KVTIER_INFLIGHT=$2 timeout 300 python scripts/trace_rt.py
done
