set -x
for cfg in c2 c3b1 c1; do
CFG=$cfg bash scripts/compare_variants.sh
GMR_TILE_ORDER=global CFG=$cfg bash scripts/compare_variants.sh
done
