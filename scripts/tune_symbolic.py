"""Nimble §3.5 symbolic-shape tuning, three steps, on one B200.

For a dense op with a symbolic token extent (Any) and static weights (N, K):
  1. tune with Any := 64: time every schedule of the space at M = 64;
  2. keep the top-k schedules of step 1 (plus the default rule);
  3. cross-evaluate the top-k on M in {1, 2, 4, ..., 256} (powers of two <= 256) and pick the
     schedule with the best average (mean over M of time / best-of-top-k time at that M).
The schedule space is the tunable part of our bf16 kernel family 1 (DISPATCH.md): the token
tile t in {32, 64, 128, 256} (the residue tile, t/16 + 1 residue variants) x the split-K
cap in {1, 2, 4, 8} = 16 schedules, plus "no schedule" (the default rule, family 4 at
M <= 128), so k = 4 here (the paper keeps 100 of AutoTVM's
thousands of template configurations; reading 23).
Held-out check: on M not used for tuning (3, 17, 48, 100, 200, 255, 384, 511) the tuned
schedule is compared with the default rule (no schedule) and with the per-M best of all 16.

Timing: a CUDA graph of 20 back-to-back nimble_dense_dyn launches (PDL chained), replayed
5x after a warm-up, CUDA events; median of 3 such runs.  Writes gpurun_out/symbolic_tuning.json
(copied to profiles/) whose "schedules" list nimble.load_dense_schedules() registers.
"""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb, synth  # noqa: E402

SHAPES = {  # (N, K) of the BERT dense ops (weights [N x K])
    "base_qkv": (2304, 768), "base_o": (768, 768), "base_ffn1": (3072, 768), "base_ffn2": (768, 3072),
    "large_qkv": (3072, 1024), "large_o": (1024, 1024), "large_ffn1": (4096, 1024), "large_ffn2": (1024, 4096),
}
# (0, 8) = no schedule: the default DISPATCH.md rule (family 4 weight streaming at one token
# tile, family 1 / 3 above) competes with the 16 family-1 schedules (round 2: the round-1 space
# predates family 4, and a schedule replaces the default rule below M = 2048)
SPACE = [(0, 8)] + list(itertools.product((32, 64, 128, 256), (1, 2, 4, 8)))
TOP_K = 4
CROSS_M = [1, 2, 4, 8, 16, 32, 64, 128, 256]
HELDOUT_M = [3, 17, 48, 100, 200, 255, 384, 511]
DEFAULT = (0, 8)


class Bench:
    def __init__(self, N, K, max_m=512, reps=20):
        self.N, self.K, self.reps = N, K, reps
        self.W = (synth.device_normal(N, K, seed=5).float() * 0.05).to(torch.bfloat16)
        self.b = torch.zeros(N, dtype=torch.float32, device="cuda")
        self.x = synth.device_normal(max_m, K, seed=6)
        self.y = torch.empty((max_m, N), dtype=torch.bfloat16, device="cuda")
        self.stream = torch.cuda.Stream()

    def time_us(self, sched, M):
        nb.set_dense_schedule(self.N, self.K, *sched)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            for _ in range(2):
                nb.dense_dyn(self.x, self.W, self.b, self.y, epi=nb.EPI_BIAS, M=M)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=self.stream):
                for _ in range(self.reps):
                    nb.dense_dyn(self.x, self.W, self.b, self.y, epi=nb.EPI_BIAS, M=M)
        runs = []
        for _ in range(3):
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            runs.append(a.elapsed_time(b) * 1e3 / (5 * self.reps))
        return sorted(runs)[1]


def tune(name, N, K):
    bench = Bench(N, K)
    step1 = {f"{t},{s}": bench.time_us((t, s), 64) for (t, s) in SPACE}
    top = sorted(SPACE, key=lambda ts: step1[f"{ts[0]},{ts[1]}"])[:TOP_K]
    if DEFAULT not in top:
        top.append(DEFAULT)          # the default rule always reaches the cross-evaluation
    step3 = {f"{t},{s}": {M: bench.time_us((t, s), M) for M in CROSS_M} for (t, s) in top}
    best_at = {M: min(step3[k][M] for k in step3) for M in CROSS_M}
    score = {k: sum(v[M] / best_at[M] for M in CROSS_M) / len(CROSS_M) for k, v in step3.items()}
    chosen = min(top, key=lambda ts: score[f"{ts[0]},{ts[1]}"])
    held = []
    for M in HELDOUT_M:
        all_t = {f"{t},{s}": bench.time_us((t, s), M) for (t, s) in SPACE}
        held.append({"M": M, "tuned_us": all_t[f"{chosen[0]},{chosen[1]}"],
                     "default_us": all_t[f"{DEFAULT[0]},{DEFAULT[1]}"], "best_of_space_us": min(all_t.values()),
                     "best_of_space": min(all_t, key=all_t.get)})
    nb.set_dense_schedule(N, K, 0, 8)
    gm = lambda xs: float(torch.tensor(xs).log().mean().exp())
    rec = {"op": name, "N": N, "K": K, "tile_t": chosen[0], "split_max": chosen[1],
           "step1_us_at_M64": step1, "top_k": [f"{t},{s}" for t, s in top], "step3_us": step3,
           "step3_avg_normalised": score, "heldout": held,
           "heldout_geomean_speedup_vs_default": gm([h["default_us"] / h["tuned_us"] for h in held]),
           "heldout_geomean_gap_to_best": gm([h["tuned_us"] / h["best_of_space_us"] for h in held])}
    print(json.dumps({k: rec[k] for k in ("op", "tile_t", "split_max", "heldout_geomean_speedup_vs_default",
                                           "heldout_geomean_gap_to_best")}), flush=True)
    return rec


def main():
    ops = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SHAPES)
    recs = [tune(op, *SHAPES[op]) for op in ops]
    out = {"procedure": "PAPER.md:392-406 three-step symbolic tuning (Any := 64, top-k, powers of two <= 256)",
           "space": [f"{t},{s}" for t, s in SPACE], "k": TOP_K, "cross_M": CROSS_M, "heldout_M": HELDOUT_M,
           "default": f"{DEFAULT[0]},{DEFAULT[1]}", "schedules": recs}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/symbolic_tuning.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
