"""Debug: where do the GPU tile lists differ from the fp32 oracle at full size?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2507_04004_b200 import rasterizer as R, scenes
from paper_2507_04004_b200.gaussians import GaussianMap
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
from test_gpu_parity import gpu_splats, _np
sc = scenes.scene_room(1 << 20, 1280, 720, lidar=32)
cam = R.camera_from(sc.cams[0])
g = GaussianMap.from_rows(sc.rows)
out = R.forward(g, cam)
m, c, cv, o, d, v = gpu_splats(out)
ent, offs, touched = O.bin_f32(m, c, cv, o, d, v, cam.width, cam.height, True)
ge = _np(out.ctx["entry_splat"]).astype(np.int64); go = _np(out.ctx["tile_offsets"]).astype(np.int64)
print("E gpu", len(ge), "oracle", len(ent))
T = len(offs) - 1
bad = 0
for t in range(T):
    a = set(ge[go[t]:go[t+1]].tolist()); b = set(ent[offs[t]:offs[t+1]].tolist())
    if a != b:
        bad += 1
        if bad <= 10:
            print("tile", t, "gpu-only", sorted(a - b)[:5], "oracle-only", sorted(b - a)[:5])
            for gid in list(a - b)[:2] + list(b - a)[:2]:
                print("   g", gid, "mean", m[gid], "conic", c[gid], "o", o[gid], "kept", int(_np(out.ctx['workspace'].view('kept','i32',(len(g),)))[gid]))
    elif not np.array_equal(ge[go[t]:go[t+1]], ent[offs[t]:offs[t+1]]):
        bad += 1
        if bad <= 10: print("tile", t, "order differs")
print("bad tiles", bad)
ws = out.ctx["workspace"]
kept = _np(ws.view("kept", "i32", (len(g),)))
rect = _np(ws.view("rect", "i32", (len(g), 4)))
cnt_o = np.bincount(ent, minlength=len(g))
cnt_g = np.bincount(ge, minlength=len(g))
diff = np.flatnonzero(cnt_o != cnt_g)
print("gaussians with different entry counts", len(diff))
for gid in diff[:12]:
    print(gid, "oracle", cnt_o[gid], "gpu", cnt_g[gid], "kept", kept[gid], "rect", rect[gid], "mean", m[gid], "conic", c[gid], "o", o[gid])
import torch
T = (cam.width + 15) // 16 * ((cam.height + 15) // 16); tw = (T + 31) // 32
mt = ws.view("huge_mask_t", "i32", (4096, tw)).cpu().numpy().view(np.uint32)
hk = np.flatnonzero(kept < 0)
bad = 0
for gid in hk:
    slot = -int(kept[gid]) - 1
    pc = int(sum(bin(int(x)).count("1") for x in mt[slot]))
    if pc != cnt_o[gid]:
        bad += 1
        if bad < 6: print("huge", gid, "slot", slot, "row popc", pc, "oracle", cnt_o[gid])
print("huge rows wrong", bad, "of", len(hk))
slots = -kept[hk] - 1
print("unique slots", len(np.unique(slots)), len(slots))
# per-Gaussian tile sets of the mismatching ones
tiles_of = {}
for gid in diff[:18]:
    tg = np.flatnonzero([gid in set(ge[go[t]:go[t+1]].tolist()) for t in range(T)]) if False else None
og_t = np.repeat(np.arange(T), np.diff(offs)); gg_t = np.repeat(np.arange(T), np.diff(go))
sel = diff[:18]
mo = np.isin(ent, sel); mg = np.isin(ge, sel)
np.savez("gpurun_out/diffdump.npz", ids=sel, s2=_np(ws.splat2d)[sel], rect=rect[sel],
         o_ent=ent[mo], o_tile=og_t[mo], g_ent=ge[mg], g_tile=gg_t[mg])
