"""Scratch: pass-1 lane utilisation of the blend backward per batch, with the
current 8x4 pixel blocks vs pixels regrouped by candidate count."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2602_14493_b200 as gmr
from oracle import gmr_oracle as orc
m = gmr.make_geodesic_sphere(158, seed=0)
cam = gmr.hemisphere_cameras(8, 3.0, (800, 800))[0]
cloud = orc.facet_gaussians(m.vertices, m.facets, np.full_like(m.vertices, 0.5))
s = orc.project(cloud, cam, np.float32)
entry, bounds = orc.bin_splats(s.mean2d, s.radius, s.depth, s.source, 800, 800)
conic = s.conic.astype(np.float64); mean = s.mean2d.astype(np.float64); op = s.opacity
ntx = 50
rng = np.random.default_rng(0)
tiles = [t for t in range(2500) if bounds[t+1]-bounds[t] > 0]
tiles = rng.choice(tiles, 150, replace=False)
yy, xx = np.mgrid[0:16, 0:16]
# warp w: 8x4 block: cols 8*(w%2).., rows 4*(w//2)..
warp_of = ((yy // 4) * 2 + (xx // 8)).ravel()
B = 100
cur_work = cur_use = srt_work = srt_use = 0
for t in tiles:
    ty, tx = divmod(t, ntx)
    ids = entry[bounds[t]:bounds[t+1]]
    px = (tx*16 + xx).ravel().astype(np.float64); py = (ty*16 + yy).ravel().astype(np.float64)
    dx = px[None, :] - mean[ids, 0:1]; dy = py[None, :] - mean[ids, 1:2]
    a, b, c = conic[ids, 0:1], conic[ids, 1:2], conic[ids, 2:3]
    power = -0.5*(a*dx*dx + c*dy*dy) - b*dx*dy
    cov = (np.minimum(0.99, op[ids, None]*np.exp(power)) >= 1/255)   # [n, 256]
    for b0 in range(0, len(ids), B):
        cnt = cov[b0:b0+B].sum(0)            # per pixel candidates in this batch
        for w in range(8):
            c_ = cnt[warp_of == w]
            cur_work += 32 * c_.max(); cur_use += c_.sum()
        srt = np.sort(cnt)
        for w in range(8):
            c_ = srt[32*w:32*w+32]
            srt_work += 32 * c_.max(); srt_use += c_.sum()
print(f"8x4 blocks: lane utilisation {cur_use/cur_work:.3f}; sorted by count: {srt_use/srt_work:.3f}")
