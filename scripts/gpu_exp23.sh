set -x
bash scripts/compare_variants.sh variants/libgmr_k5m5.so variants/libgmr_k5m5a2.so variants/libgmr_k5a8.so
CFG=c3b1 bash scripts/compare_variants.sh variants/libgmr_k5m5.so
