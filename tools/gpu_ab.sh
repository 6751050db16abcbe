#!/bin/bash
# A/B variants of libgslic.so on one box: bench it/s and a warm graph-replay kernel list each.
#   gpurun --timeout 1200 -- bash tools/gpu_ab.sh <tag> base "name:DEF1,DEF2" ...
# AB_TEST=1: also run the GPU test suite against each variant.
# "name@VAR=v,VAR2=w": the in-tree build run with those environment variables.
# "base" = the in-tree build; other entries are built with -D flags into lib/var_<name>.so.
TAG=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build_$TAG.log 2>&1
for spec in "$@"; do
  envs=""
  if [[ "$spec" == *@* ]]; then envs=$(echo "${spec#*@}" | tr ',' ' '); spec="${spec%%@*}:"; fi
  name=${spec%%:*}; defs=${spec#*:}
  if [ "$name" = "base" ] || [ -z "$defs" ]; then lib=""; else
    lib=$PWD/paper_2507_04004_b200/lib/var_$name.so
    args=$(echo "$defs" | tr ',' '\n' | sed 's/^/-D/' | tr '\n' ' ')
    python -m paper_2507_04004_b200.build $args --out=$lib >> gpurun_out/ab_build_$TAG.log 2>&1 || echo "build $name failed"
  fi
  if [ -n "$AB_TEST" ] && [ "$name" != "base" ]; then
    env $envs GSLIC_LIB=$lib timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ab_${TAG}_${name}_pt.log 2>&1
    echo "$name pytest: $(tail -1 gpurun_out/ab_${TAG}_${name}_pt.log)"
  fi
  env $envs GSLIC_LIB=$lib timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_${TAG}_$name.json 2> gpurun_out/ab_${TAG}_$name.err
  env $envs GSLIC_LIB=$lib timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --cache-control none --csv --log-file gpurun_out/ab_${TAG}_$name.csv \
    python tools/prof_graph.py S2r-1M-1280x720-32line 8 > /dev/null 2>&1
  echo "$name $(python -c "import json;d=json.load(open('gpurun_out/ab_${TAG}_$name.json'));print(d['value'], d['e2e']['value'])" 2>&1)"
  python tools/graph_table.py gpurun_out/ab_${TAG}_$name.csv 8 2>&1 | sed -n 5,10p
done
