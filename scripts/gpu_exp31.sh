bash scripts/compare_variants.sh > /dev/null 2>&1
GMR_TILE_ORDER=global bash scripts/compare_variants.sh > /dev/null 2>&1
CFG=c2 bash scripts/compare_variants.sh > /dev/null 2>&1
GMR_TILE_ORDER=global CFG=c2 bash scripts/compare_variants.sh > /dev/null 2>&1
cat gpurun_out/variants.txt | cut -c1-170
