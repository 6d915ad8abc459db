# final 1-GPU check: full GPU suite, smoke, default bench
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err
python -c "import json; d=json.loads(open('gpurun_out/bench_final.json').read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['gpu_launches'], d.get('other_arith',{}).get('value'))"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_final.json 2> /dev/null; cat gpurun_out/ref_final.json | cut -c 1-300
