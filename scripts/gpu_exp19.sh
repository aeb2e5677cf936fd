set -x
bash scripts/compare_variants.sh
GMR_TILE_ORDER=global bash scripts/compare_variants.sh
