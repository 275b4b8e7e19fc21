#!/bin/bash
# A/B timing of experimental builds: prints K1..K6 stage ms per step for each.
for d in "$@"; do
  if [ "$d" = "main" ]; then unset SSB_LIB_PATH; else export SSB_LIB_PATH=$PWD/paper_2603_20481_b200/$d/libspecsense_b200.so; fi
  python bench.py --no-cpu --no-e2e --steps 5 $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', round(d['value']), {k: round(v,3) for k,v in d['stage_ms_per_step'].items()})"
done
