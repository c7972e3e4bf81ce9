python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "model" > gpurun_out/model.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/model.log
timeout 900 python bench.py --steps 16 --warmup 4 > gpurun_out/bench_m.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads([l for l in open('gpurun_out/bench_m.log') if l.startswith('{')][-1]);print(d['value'], d['model_decode'])"
tail -5 gpurun_out/bench_m.log | cut -c1-300
