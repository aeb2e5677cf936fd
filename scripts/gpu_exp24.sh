set -x
timeout 900 python -m pytest tests/test_gpu_fit.py -x -q -s > gpurun_out/tests_fit.log 2>&1; tail -8 gpurun_out/tests_fit.log
timeout 600 python bench.py --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 700 gpurun_out/bench_c5.json
