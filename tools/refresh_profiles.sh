#!/bin/bash
# round-1 refresh: bench lines, reference arm, launch list, ncu full captures
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r01_bench_c5r.json 2> gpurun_out/bench_c5r.err; echo c5r=$?
timeout 600 python bench.py --mode c5r16 > gpurun_out/r01_bench_c5r16.json 2> gpurun_out/bench_c5r16.err; echo c5r16=$?
timeout 600 python bench.py --mode hann > gpurun_out/r01_bench_hann.json 2> gpurun_out/bench_hann.err; echo hann=$?
timeout 900 python bench.py --impl reference > gpurun_out/r01_reference_arm.json 2> gpurun_out/ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv bash tools/prof_cmd.sh > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fft_mag_kernel -c 1 -o gpurun_out/k1_full bash tools/prof_cmd.sh > gpurun_out/ncu_k1.log 2>&1; echo k1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:binarize_tile -c 1 -o gpurun_out/k4_full bash tools/prof_cmd.sh > gpurun_out/ncu_k4.log 2>&1; echo k4=$?
