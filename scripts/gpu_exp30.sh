set -x
GMR_LIB_PATH=$PWD/variants/libgmr_f64rec.so timeout 900 python -m pytest tests -m gpu -x -q -k "parity or stress or configs or fullsize or edges" > gpurun_out/tests_f64rec.log 2>&1; tail -2 gpurun_out/tests_f64rec.log
timeout 300 python scripts/f64_stages.py f64
GMR_LIB_PATH=$PWD/variants/libgmr_f64rec.so timeout 300 python scripts/f64_stages.py f64
