set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_lb.log 2>&1; tail -2 gpurun_out/tests_lb.log
for cfg in c3 c4 c3b1 c1; do CFG=$cfg bash scripts/compare_variants.sh; done
GMR_TILE_ORDER=global bash scripts/compare_variants.sh
