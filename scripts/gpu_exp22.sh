set -x
GMR_LIB_PATH=$PWD/variants/libgmr_cov2.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_cov2.log 2>&1; tail -2 gpurun_out/tests_cov2.log
bash scripts/compare_variants.sh variants/libgmr_cov2.so
