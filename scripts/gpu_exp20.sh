set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_kr.log 2>&1; tail -2 gpurun_out/tests_kr.log
bash scripts/compare_variants.sh
GMR_TILE_ORDER=global bash scripts/compare_variants.sh
CFG=c4 bash scripts/compare_variants.sh
