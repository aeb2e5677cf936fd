# ncu --set full of K1 (mesh_to_splats) and K5 (face_views_backward), one launch each, config 3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"mesh_to_splats|face_views_backward" -s 4 -c 2 \
  -o gpurun_out/k1k5 -f python bench.py --config c3 --steps 1 --warmup 3 --no-cpu --no-extras > gpurun_out/ncu_k1k5.log 2>&1
tail -2 gpurun_out/ncu_k1k5.log
