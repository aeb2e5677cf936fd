set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or edges or stress or configs" > gpurun_out/tests_dsb3.log 2>&1; tail -2 gpurun_out/tests_dsb3.log
bash scripts/compare_variants.sh
CFG=c4 bash scripts/compare_variants.sh
