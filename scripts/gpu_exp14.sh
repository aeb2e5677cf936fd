set -x
GMR_LIB_PATH=$PWD/variants/libgmr_k5s.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or configs or fullsize or stress" > gpurun_out/tests_k5s.log 2>&1; tail -2 gpurun_out/tests_k5s.log
bash scripts/compare_variants.sh variants/libgmr_k5s.so variants/libgmr_k5s1536.so variants/libgmr_k5s1024.so variants/libgmr_k5s3072.so
