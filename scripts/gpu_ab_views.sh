set -x
for so in paper_2602_14493_b200/libgmr.so variants/libgmr_prev.so variants/libgmr_nopin.so paper_2602_14493_b200/libgmr.so; do
  for cfg in views c1; do
    GMR_LIB_PATH=$PWD/$so timeout 600 python bench.py --config $cfg --no-cpu > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print(sys.argv[1], sys.argv[2], d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'))" $so $cfg >> gpurun_out/ab.txt
  done
done
cat gpurun_out/ab.txt
