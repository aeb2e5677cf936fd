set -x
bash scripts/compare_variants.sh variants/libgmr_fw96.so variants/libgmr_fw64.so variants/libgmr_fw128.so
GMR_LIB_PATH=$PWD/variants/libgmr_fw96.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_fw96.log 2>&1; tail -3 gpurun_out/tests_fw96.log
