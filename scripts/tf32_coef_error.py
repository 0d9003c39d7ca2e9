"""CPU experiment: image error when the coef operand is rounded to tf32 (the
reason pass B keeps the 3xTF32 hi/lo split).  python scripts/tf32_coef_error.py"""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
import oracle.rfsplat_oracle as O
def tf32_rn(x):
    x = np.asarray(x, np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    b = ((b + 0x1000) & 0xFFFFE000).astype(np.uint32)   # round half up on the 13 dropped bits
    return b.view(np.float32)
for n, F in [(20000, 52), (4000, 1), (16000, 8)]:
    c = O.round_f32(O.bench_scene(n, F=F))
    for seed in (1000, 7):
        tx = O.sample_tx(seed, 1)[0]
        pr = O.prepare(c, np.zeros(3), np.eye(3), tx, 360, 90)
        bins = O.tile_bins(pr)
        coef = (pr.s / pr.d_tx[:, None]).astype(np.float32)
        ct = tf32_rn(coef)
        worst = 0; mx = 0
        for key in sorted(bins):
            ys, xs = O._tile_px(key[0], key[1], 360, 90)
            rows = bins[key]
            gx, gy = np.meshgrid((xs+0.5).astype(np.float32), (ys+0.5).astype(np.float32))
            a = O._alphas(pr, rows, gx.ravel(), gy.ravel(), np.float32)[0]
            om = 1-a; tb = np.ones_like(a); tb[1:] = np.cumprod(om[:-1], axis=0)
            act = (tb >= 1e-4) & (a > 0)
            wgt = np.where(act, tb*a, 0).astype(np.float64)
            ref = wgt.T @ coef[rows].astype(np.float64)
            got = wgt.T @ ct[rows].astype(np.float64)
            worst = max(worst, np.abs(got-ref).max()); mx = max(mx, np.abs(ref).max())
        print(n, F, seed, 'normwise err tf32 coef:', worst/mx)
