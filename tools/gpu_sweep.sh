#!/bin/bash
# gpurun --timeout 2400 -- bash tools/gpu_sweep.sh <tag>: bench line of every BASELINE config
# that fits one GPU (500k / 1M training, LiDAR density sweep, 2M 1080p render FPS, S1 stress)
TAG=${1:-sw}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
: > gpurun_out/sweep_$TAG.jsonl
for C in S2r-500k-1280x720-32line S2r-1M-1280x720-32line S2r-1M-1280x720-16line S2r-1M-1280x720-64line \
         S2r-1M-1280x720-128line S2r-1M-1280x720-livox5k S2r-1M-1280x720-livox200k S2r-2M-1920x1080-render S2r-1M-1280x720-track \
         S1-1M-1280x720 S1-10k-320x240; do
  timeout 600 python bench.py --config $C --steps 300 --warmup 5 --no-cpu-baseline >> gpurun_out/sweep_$TAG.jsonl \
      2>> gpurun_out/sweep_$TAG.err
done
# the reference arm (float64 CPU oracle, all host cores) for the render and tracking configs
for C in S2r-2M-1920x1080-render S2r-1M-1280x720-track; do
  timeout 600 python bench.py --impl reference --config $C --steps 2 --warmup 0 >> gpurun_out/sweep_$TAG.jsonl \
      2>> gpurun_out/sweep_$TAG.err
done
python - "$TAG" <<'PY'
import json, sys
for l in open(f"gpurun_out/sweep_{sys.argv[1]}.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], d.get("impl", "ours"), d["value"], d["unit"], (d.get("e2e") or {}).get("value"))
PY
