set -x
GMR_LIB_PATH=$PWD/variants/libgmr_skip0.so timeout 900 python -m pytest tests -m gpu -x -q -k "parity or stress or configs or fullsize" > gpurun_out/tests_skip0.log 2>&1; tail -2 gpurun_out/tests_skip0.log
bash scripts/compare_variants.sh variants/libgmr_skip0.so
