#!/bin/bash
# One config-5-as-written step set for profiling (same command with and without ncu).
python bench.py --mode hann --batch 296 --steps 2 --warmup 1 --no-cpu --e2e-batch 2 --distinct 4
