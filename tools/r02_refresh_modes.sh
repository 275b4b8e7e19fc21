cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python bench.py --mode hann > gpurun_out/r02_bench_hann.json 2> gpurun_out/hann.err; echo hann=$?
timeout 900 python bench.py --mode c5r16 > gpurun_out/r02_bench_c5r16.json 2> gpurun_out/c5r16.err; echo c5r16=$?
timeout 900 python bench.py --mode stream > gpurun_out/r02_bench_stream.json 2> gpurun_out/stream.err; echo stream=$?
timeout 900 python bench.py --mode stream5 > gpurun_out/r02_bench_stream5.json 2> gpurun_out/stream5.err; echo stream5=$?
