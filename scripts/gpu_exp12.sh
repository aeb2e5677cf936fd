set -x
for v in tma tmap2; do
GMR_LIB_PATH=$PWD/variants/libgmr_$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "parity or edges or stress or configs or fullsize" > gpurun_out/tests_$v.log 2>&1; tail -2 gpurun_out/tests_$v.log
done
bash scripts/compare_variants.sh variants/libgmr_tma0.so variants/libgmr_tma.so variants/libgmr_p2.so variants/libgmr_tmap2.so
