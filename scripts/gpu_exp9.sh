set -x
for v in lsort lsortb; do
GMR_LIB_PATH=$PWD/variants/libgmr_$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or edges or stress or configs" > gpurun_out/tests_$v.log 2>&1; tail -3 gpurun_out/tests_$v.log
done
bash scripts/compare_variants.sh variants/libgmr_lsort.so variants/libgmr_lsortb.so
