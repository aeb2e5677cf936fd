# compute-sanitizer passes over small invocations of every blend / binning path
# (one B200): memcheck on smoke(), racecheck + synccheck on a small render
set -x
mkdir -p gpurun_out/san
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/memcheck_smoke.log 2>&1; echo "memcheck smoke $?"
tail -5 gpurun_out/san/memcheck_smoke.log
cat > /tmp/san_small.py <<'PY'
import numpy as np, torch
import paper_2602_14493_b200 as gmr
from paper_2602_14493_b200 import engine
m = gmr.make_icosphere(1280)
mesh = gmr.TriangleMesh(m.vertices, m.facets, gmr.seeded_colors(m.num_vertices, 0))
cams = gmr.hemisphere_cameras(2, 3.0, (96, 80))
dev = torch.device("cuda", 0)
pos = torch.tensor(np.asarray(mesh.vertices), dtype=torch.float32, device=dev)
col = torch.tensor(np.asarray(mesh.colors), dtype=torch.float32, device=dev)
faces = torch.tensor(np.asarray(mesh.facets), dtype=torch.int32, device=dev)
for flags in (0, engine.lib.FLAG_TILE_DEPTH_SORT):
    rgb, alpha, st = engine.render_forward(pos, col, faces, cams, 96, 80, (0.1, 0.1, 0.1), flags=flags)
    g = torch.randn_like(rgb); ga = torch.randn_like(alpha)
    engine.render_backward(st, pos, col, faces, rgb, g, ga)
torch.cuda.synchronize()
print("ok")
PY
for tool in racecheck synccheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_small.py > gpurun_out/san/${tool}_small.log 2>&1; echo "$tool small $?"
  tail -4 gpurun_out/san/${tool}_small.log
done
