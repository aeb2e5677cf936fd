set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_pdl.log 2>&1; tail -2 gpurun_out/tests_pdl.log
for cfg in c3 c1 c3b1; do
  CFG=$cfg bash scripts/compare_variants.sh
  GMR_PDL=0 CFG=$cfg bash scripts/compare_variants.sh
done
timeout 300 python scripts/c5_loop_check.py
GMR_PDL=0 timeout 300 python scripts/c5_loop_check.py
