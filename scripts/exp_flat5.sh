KVT_FLAT_TRACE=1 python -c "import paper_2605_09490_b200.build as b; b.build(force=True)" 
TAG=base timeout 300 python scripts/trace_rt.py
TAG=nopf KVTIER_L2PF_MB=0 timeout 300 python scripts/trace_rt.py
TAG=pf8 KVTIER_L2PF_MB=8 timeout 300 python scripts/trace_rt.py
TAG=fv2_nopf KVTIER_FVAR=2 KVTIER_L2PF_MB=0 timeout 300 python scripts/trace_rt.py
TAG=fv4_nopf KVTIER_FVAR=4 KVTIER_L2PF_MB=0 timeout 300 python scripts/trace_rt.py
