python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for C in S1-1M-1280x720 S2r-1M-1280x720-32line S1-10k-320x240; do timeout 300 python bench.py --config $C --steps 300 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['config']['workload'], d['value'], d['e2e']['value'] if d.get('e2e') else None)"; done
