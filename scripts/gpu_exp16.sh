set -x
bash scripts/compare_variants.sh variants/libgmr_dsb.so
CFG=c4 bash scripts/compare_variants.sh variants/libgmr_dsb.so
