"""Per-k-block timeline of CTA 0 of one dense_dyn launch (NIMBLE_DBG=4 + nimble_debug_trace):
when the MMA thread sees each stage full, when the producer sees each stage empty, and when
each tile's accumulator is free.  Intervals vs the k-block's nominal MMA time show whether
the tensor pipe is fed (MMA-bound: full-to-full ~ MMA time) or starved."""
import os
import sys

import numpy as np
import torch

os.environ["NIMBLE_DBG"] = "4"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb  # noqa: E402

for shp in (sys.argv[1] if len(sys.argv) > 1 else "17448x3072x1024,17448x1024x4096").split(","):
    M, N, K = (int(v) for v in shp.split("x"))
    W = torch.randn((N, K), device="cuda", dtype=torch.bfloat16) * 0.02
    b = torch.zeros((N,), device="cuda", dtype=torch.float32)
    x = torch.randn((M, K), device="cuda", dtype=torch.bfloat16)
    y = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        nb.dense_dyn(x, W, b, y)
    torch.cuda.synchronize()
    buf = torch.zeros(32768 + 4 * 512, dtype=torch.int64, device="cuda")
    nb._lib.nimble_debug_trace(buf.data_ptr())
    nb.dense_dyn(x, W, b, y)
    torch.cuda.synchronize()
    nb._lib.nimble_debug_trace(None)
    t = buf.cpu().numpy().astype(np.float64)
    full = t[8192:8192 + 4096]
    full = full[full > 0]
    empty = t[16384:16384 + 4096]
    empty = empty[empty > 0]
    tiles = t[24576:24576 + 256]
    tiles = tiles[tiles > 0]
    d = nb.last_dispatch()
    kd = 2 if (K % 64 == 0 and K >= 128 and os.environ.get("NIMBLE_KD") != "1") else 1
    kb = ((K + 63) // 64 + kd - 1) // kd                 # pipeline stages per tile (kd k-blocks each)
    df = np.diff(full)
    print(f"{shp}: family {d['family']} t={d['tile_t']} stages/tile={kb} (kd={kd}); CTA 0: {len(full)} stages, {len(tiles)} tiles")
    print("  MMA full->full interval clk: median %.0f  p10 %.0f  p90 %.0f  max %.0f  (nominal MMA per stage @8192 flop/clk/SM: %d)"
          % (np.median(df), np.percentile(df, 10), np.percentile(df, 90), df.max(), kd * 256 * d["tile_t"] * 64 * 2 // 2 // 8192))
    if len(empty) > 1:
        de = np.diff(empty)
        print("  producer empty->empty interval clk: median %.0f  p90 %.0f" % (np.median(de), np.percentile(de, 90)))
    within = [df[i] for i in range(len(df)) if (i + 1) % kb != 0]
    across = [df[i] for i in range(len(df)) if (i + 1) % kb == 0]
    print("  within-tile median %.0f, tile-boundary median %.0f" % (np.median(within), np.median(across) if across else -1))
    print("  first 24 intervals:", " ".join("%d" % v for v in df[:24]))
    pos = np.arange(len(df)) % kb                    # interval i ends at k-block i+1
    prof = [np.mean(df[pos == q]) for q in range(min(kb, 16)) if np.any(pos == q)]
    print("  mean interval by k-block position in tile (first 16):", " ".join("%d" % v for v in prof))
    print("  mean %.0f; share of time in intervals > 800 clk: %.0f%%" % (df.mean(), 100 * df[df > 800].sum() / df.sum()))
    g1, g2 = [], []
    for i in range(1, min(len(tiles), len(full) // kb)):
        g1.append(tiles[i] - full[i * kb - 1])          # last full of tile i-1 -> accumulator free
        g2.append(full[i * kb] - tiles[i])              # accumulator free -> first full of tile i
    if g1:
        print("  tile boundary: last k-block -> acc free median %.0f; acc free -> first full median %.0f"
              % (np.median(g1), np.median(g2)))
    ph = t[:148 * 8].reshape(148, 8)                # per-CTA globaltimer ns: 0 start, 1 setup, 2 first data, 6 end
    ok = ph[:, 0] > 0
    t0 = ph[ok, 0].min()
    print("  CTA phases (us from first CTA start): start max %.2f; setup done med %.2f; first data med %.2f max %.2f;"
          " end med %.2f max %.2f" % ((ph[ok, 0].max() - t0) / 1e3, (np.median(ph[ok, 1]) - t0) / 1e3,
                                     (np.median(ph[ok, 2]) - t0) / 1e3, (ph[ok, 2].max() - t0) / 1e3,
                                     (np.median(ph[ok, 6]) - t0) / 1e3, (ph[ok, 6].max() - t0) / 1e3))
    ep = t[32768:32768 + 4 * 512].reshape(-1, 4)
    ep = ep[ep[:, 0] > 0]
    if len(ep) > 1:
        print("  epilogue per tile (clk): acc ready -> staged median %.0f; staged -> store drained %.0f;"
              " acc-ready to acc-ready %.0f; MMA tile (full 0 -> full 0) %.0f"
              % (np.median(ep[:, 1] - ep[:, 0]), np.median(ep[:, 2] - ep[:, 1]), np.median(np.diff(ep[:, 0])),
                 np.median(np.diff(full[::kb])) if len(full) > kb else -1))
        # does the MMA wait for the accumulator? tile i's acc-free vs epilogue of tile i-2 staged
        lag = [tiles[i] - ep[i - 2, 1] for i in range(2, min(len(tiles), len(ep) + 2))]
        print("  MMA acc-free minus epilogue(i-2) staged (clk, >0 = MMA could proceed only after it): median %.0f"
              % np.median(lag))
    clk = t[30002] - t[30000]
    ns = t[30003] - t[30001]
    print("  CTA 0 SM clock over its k-blocks: %.0f MHz (%.0f clk in %.1f us)" % (1e3 * clk / max(ns, 1), clk, ns / 1e3))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(20):
        nb.dense_dyn(x, W, b, y)
    ev1.record()
    torch.cuda.synchronize()
    print("  stream-timed per launch (20 back to back, host enqueue): %.2f us" % (ev0.elapsed_time(ev1) * 1e3 / 20))
