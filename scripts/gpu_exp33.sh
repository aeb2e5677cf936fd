for cfg in c3 c4; do CFG=$cfg bash scripts/compare_variants.sh variants/libgmr_binw.so > /dev/null 2>&1; done
cat gpurun_out/variants.txt | cut -c1-150
