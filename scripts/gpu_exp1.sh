set -x
bash profiles/pair_sol/run.sh > gpurun_out/pair_sol.txt 2>&1; cat gpurun_out/pair_sol.txt
bash scripts/compare_variants.sh variants/libgmr_b128m4.so variants/libgmr_b256k48m3.so variants/libgmr_b256k40m4.so
