set -x
bash scripts/compare_variants.sh variants/libgmr_fnb.so variants/libgmr_fnbcm.so
GMR_LIB_PATH=$PWD/variants/libgmr_fnbcm.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or edges or configs" > gpurun_out/tests_fnbcm.log 2>&1; tail -3 gpurun_out/tests_fnbcm.log
