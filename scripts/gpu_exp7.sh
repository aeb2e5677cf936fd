set -x
bash scripts/compare_variants.sh variants/libgmr_pin.so variants/libgmr_pinb.so
