set -x
GMR_LIB_PATH=$PWD/variants/libgmr_trig.so timeout 900 python -m pytest tests -m gpu -x -q -k "parity or stress or configs or fullsize or torch_api or fit" > gpurun_out/tests_trig.log 2>&1; tail -2 gpurun_out/tests_trig.log
for cfg in c3 c3b1 c1; do
  CFG=$cfg bash scripts/compare_variants.sh variants/libgmr_trig.so
done
timeout 300 python scripts/c5_loop_check.py
GMR_LIB_PATH=$PWD/variants/libgmr_trig.so timeout 300 python scripts/c5_loop_check.py
