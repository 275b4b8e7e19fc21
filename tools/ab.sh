#!/bin/bash
# A/B timing of experimental builds (tools/variant.py): prints K1..K6 stage ms
# per step for each build, in the order given, twice (order effects).
for pass in 1 2; do
for d in "$@"; do
  if [ "$d" = "main" ]; then unset SSB_LIB_PATH; else export SSB_LIB_PATH=$PWD/paper_2603_20481_b200/$d/libspecsense_b200.so; fi
  python bench.py --no-cpu --no-e2e --no-hann --no-verify --steps ${STEPS:-10} $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms_per_step'].items()})"
done
done
