timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests_gi.log 2>&1; tail -1 gpurun_out/tests_gi.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in c3 c3b1 c2; do CFG=$cfg bash scripts/compare_variants.sh > /dev/null 2>&1; done
cat gpurun_out/variants.txt | cut -c1-150
