set -x
GMR_LIB_PATH=$PWD/variants/libgmr_k5r.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or configs or fullsize" > gpurun_out/tests_k5r.log 2>&1; tail -2 gpurun_out/tests_k5r.log
GMR_LIB_PATH=$PWD/variants/libgmr_atomic.so timeout 600 python -m pytest tests -m gpu -q -k "parity or configs or fullsize" > gpurun_out/tests_atomic.log 2>&1; tail -2 gpurun_out/tests_atomic.log
bash scripts/compare_variants.sh variants/libgmr_base2.so variants/libgmr_atomic.so variants/libgmr_k5r.so variants/libgmr_k5r8a8.so
