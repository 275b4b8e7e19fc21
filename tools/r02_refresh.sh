#!/bin/bash
# round-2 refresh: GPU tests, default bench line, reference arm, launch list,
# ncu full captures of K1 / K4 / K5+K6 (summaries go to profiles/r02_*)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.txt 2>&1; echo gputest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.txt 2>&1; echo smoke=$?
fi
timeout 900 python bench.py > gpurun_out/r02_bench_c5r.json 2> gpurun_out/bench_c5r.err; echo c5r=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02_reference_arm.json 2> gpurun_out/ref.err; echo ref=$?
[ "${SKIP_NCU:-0}" = 1 ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv bash tools/prof_cmd.sh > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fft_mag_kernel -c 1 -o gpurun_out/r02_k1_full bash tools/prof_cmd.sh > gpurun_out/ncu_k1.log 2>&1; echo k1=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:binarize_tile -c 1 -o gpurun_out/r02_k4_full bash tools/prof_cmd.sh > gpurun_out/ncu_k4.log 2>&1; echo k4=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"floor_kernel|consolidate_kernel|count_runs|scan_rows|plot_base|emit_runs|union_block|union_boundary|flatten|compact_kernel" -c 10 -o gpurun_out/r02_k3k5k6_full bash tools/prof_cmd.sh > gpurun_out/ncu_k5k6.log 2>&1; echo k3k5k6=$?
