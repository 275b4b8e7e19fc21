#!/bin/bash
# One fused-pipeline step set for profiling (same command with and without ncu).
python bench.py --batch 296 --steps 2 --warmup 1 --no-cpu --e2e-batch 2 --distinct 4
