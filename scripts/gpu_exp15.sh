set -x
GMR_LIB_PATH=$PWD/variants/libgmr_wg.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or configs or fullsize or stress or torch_api" > gpurun_out/tests_wg.log 2>&1; tail -2 gpurun_out/tests_wg.log
bash scripts/compare_variants.sh variants/libgmr_wg.so
