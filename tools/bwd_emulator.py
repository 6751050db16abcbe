"""Diagnostic (test infrastructure): numpy emulation of the device blend + backward
(render.cu) with a selectable precision per stage, to find which fp32 operation limits the
parameter-gradient parity of near-camera Gaussians against the float64 reference.

    python tools/bwd_emulator.py [scene]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

f32, f64 = np.float32, np.float64


def normwise(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-12))


def run(z, P):
    """P: dict of stage -> dtype ('alpha', 'state', 'terms', 'sum')."""
    cam = O.Camera(int(z["width"]), int(z["height"]), float(z["fx"]), float(z["fy"]), float(z["cx"]),
                   float(z["cy"]), z["rot_cw"], z["trans_cw"])
    rows = z["rows"].astype(f32).astype(f64)
    g = O.GaussianMap.from_rows(rows)
    out = O.forward(g, cam)
    proj, ctx = out.ctx["proj"], out.ctx
    c = proj["conic"]
    a64, b64, c64 = c[:, 0], c[:, 1], c[:, 2]
    ok = a64 > 0
    A = a64.astype(f32)
    beta = np.where(ok, b64 / np.where(ok, a64, 1), 0).astype(f32)
    gam = np.where(ok, (a64 * c64 - b64 * b64) / np.where(ok, a64, 1), 0).astype(f32)
    mx, my = proj["mean2d"][:, 0].astype(f32), proj["mean2d"][:, 1].astype(f32)
    op = ctx["opac"].astype(f32)
    dep = proj["depth"].astype(f32)
    col = ctx["colors"].astype(f32)
    ent, offs = ctx["entry_splat"], ctx["tile_offsets"]
    W, H = cam.width, cam.height
    tx_n = (W + 15) // 16
    gc = z["g_color"].astype(f32)
    gd = z["g_depth"].astype(f32)
    go = z["g_opac"].astype(f32)
    n = len(rows)
    g2d = np.zeros((n, 10))
    ta, ts, tt = P["alpha"], P["state"], P["terms"]

    def alpha_of(gi, fx, fy):
        dx = (fx - mx[gi]).astype(f32)
        dy = (fy - my[gi]).astype(f32)
        u = (beta[gi].astype(f64) * dy + dx).astype(ta)  # fma: one rounding
        au = (ta(A[gi]) * u).astype(ta)
        q = (au.astype(f64) * u + (ta(gam[gi]) * dy * dy).astype(f64)).astype(ta)
        e = np.exp(ta(-0.5) * q).astype(ta)
        araw = (ta(op[gi]) * e).astype(ta)
        clamped = araw > ta(0.99)
        alpha = np.where(clamped, ta(0.99), araw).astype(ta)
        om = np.where(clamped, ta(0.01), (1.0 - op[gi].astype(f64) * e).astype(ta)).astype(ta)
        return dx, dy, au, e, alpha, om, clamped

    for t in range(len(offs) - 1):
        s, e_ = int(offs[t]), int(offs[t + 1])
        if s == e_:
            continue
        ty, tx = divmod(t, tx_n)
        ys, xs = np.mgrid[ty * 16:min(ty * 16 + 16, H), tx * 16:min(tx * 16 + 16, W)]
        fx, fy = xs.ravel().astype(f32), ys.ravel().astype(f32)
        pix = (ys.ravel(), xs.ravel())
        # forward (fp32 state as the device; alpha in the chosen precision)
        T = np.ones(len(fx), ta)
        cnt = np.zeros(len(fx), int)
        done = np.zeros(len(fx), bool)
        for k in range(s, e_):
            gi = ent[k]
            *_, alpha, om, _ = alpha_of(gi, fx, fy)
            live = ~done
            T = np.where(live, (T * om).astype(ta), T)
            cnt = np.where(live, k - s + 1, cnt)
            done = done | (live & (T < 1e-4))
            if done.all():
                break
        # backward: back-to-front replay from the final T
        Tb_state = T.astype(ts)
        S = np.zeros((len(fx), 5), ts)
        gcp, gdp, gop = gc[pix].astype(ts), gd[pix].astype(ts), go[pix].astype(ts)
        mc = cnt.max()
        for k in range(s + mc - 1, s - 1, -1):
            le = k - s
            act = le < cnt
            gi = ent[k]
            dx, dy, au, e, alpha, om, clamped = alpha_of(gi, fx, fy)
            rom = (ts(1.0) / om.astype(ts)).astype(ts)
            Tb = (Tb_state * rom).astype(ts)
            w = (alpha.astype(ts) * Tb).astype(ts)
            cvec = col[gi].astype(ts)
            dl = (Tb * ((cvec[0] * gcp[:, 0] + cvec[1] * gcp[:, 1] + cvec[2] * gcp[:, 2]) + ts(dep[gi]) * gdp + gop)
                  - (S[:, 0] * gcp[:, 0] + S[:, 1] * gcp[:, 1] + S[:, 2] * gcp[:, 2] + S[:, 3] * gdp + S[:, 4] * gop)
                  * rom).astype(ts)
            gq = (dl.astype(tt) * (tt(-0.5) * alpha.astype(tt))).astype(tt)
            v = np.zeros((len(fx), 10))
            nc = ~clamped & act
            v[:, 0] = np.where(nc, gq * (tt(-2) * au.astype(tt)), 0)
            v[:, 1] = np.where(nc, gq * (tt(-2) * (tt(beta[gi]) * au.astype(tt) + tt(gam[gi]) * dy.astype(tt))), 0)
            v[:, 2] = np.where(nc, gq * dx.astype(tt) * dx.astype(tt), 0)
            v[:, 3] = np.where(nc, gq * tt(2) * dx.astype(tt) * dy.astype(tt), 0)
            v[:, 4] = np.where(nc, gq * dy.astype(tt) * dy.astype(tt), 0)
            v[:, 5] = np.where(nc, dl.astype(tt) * e.astype(tt), 0)
            v[:, 6:9] = np.where(act[:, None], w[:, None] * gcp[:, :3], 0)
            v[:, 9] = np.where(act, w * gdp, 0)
            if P["sum"] == "pair":  # device: 2 pixels (rows y, y + 8) per thread in fp32, the rest in f64
                vv = v.astype(f32)
                nr = len(vv) // 16
                if nr == 16:
                    vv = vv.reshape(2, 8 * 16, 10)
                    vv = (vv[0] + vv[1]).astype(f32)
                g2d[gi] += vv.astype(f64).sum(axis=0)
            else:
                g2d[gi] += v.astype(P["sum"]).sum(axis=0, dtype=P["sum"])
            upd = act
            S[:, 0:3] = np.where(upd[:, None], (S[:, 0:3] + cvec[None, :] * w[:, None]).astype(ts), S[:, 0:3])
            S[:, 3] = np.where(upd, (S[:, 3] + ts(dep[gi]) * w).astype(ts), S[:, 3])
            S[:, 4] = np.where(upd, (S[:, 4] + w).astype(ts), S[:, 4])
            Tb_state = np.where(upd, Tb, Tb_state)
    touched = np.zeros(n, bool)
    touched[ent] = True
    grows = O.chain(rows, cam, g2d, touched)
    return grows, g2d


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "room4096"
    z = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    groups = {"pos": (0, 3), "ls": (3, 6), "quat": (6, 10), "op": (10, 11)}
    for label, P in [("all f64", dict(alpha=f64, state=f64, terms=f64, sum=f64)),
                     ("alpha f32", dict(alpha=f32, state=f64, terms=f64, sum=f64)),
                     ("state f32", dict(alpha=f64, state=f32, terms=f64, sum=f64)),
                     ("terms f32", dict(alpha=f64, state=f64, terms=f32, sum=f64)),
                     ("sum f32", dict(alpha=f64, state=f64, terms=f64, sum=f32)),
                     ("all f32", dict(alpha=f32, state=f32, terms=f32, sum=f32)),
                     ("f32+pair", dict(alpha=f32, state=f32, terms=f32, sum="pair")),
                     ("f32+f64sum", dict(alpha=f32, state=f32, terms=f32, sum=f64))]:
        gr, _ = run(z, P)
        print(f"{label:10s}", " ".join(f"{k}:{normwise(gr[:, a:b], z['grads'][:, a:b]):.1e}" for k, (a, b) in groups.items()),
              flush=True)


if __name__ == "__main__":
    main()
