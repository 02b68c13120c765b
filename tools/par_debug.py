"""Parity debug of the bench loop: two layer buffers decoded alternately as in
bench.py (no timing), unit 0 of buffer 0 recorded after every step, then the
C oracle replays the same steps and every step is compared; a second GPU pass
over identical inputs checks run-to-run determinism."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from oracle import oracle as O
from paper_2505_02922_b200 import EngineConfig, WaveLayer
dev = torch.device("cuda")
U, G, d, n = int(os.environ.get("U", 128)), int(os.environ.get("G", 4)), 128, int(os.environ.get("N", 122880))
NB, STEPS = int(os.environ.get("NB", 2)), int(os.environ.get("STEPS", 40))
UPD = os.environ.get("UPD") == "1"
EST_FRAC = float(os.environ.get("EST_FRAC", 0.232))
RET_FRAC = float(os.environ.get("RET_FRAC", 0.018))  # decode() with index updates (STEPS past the first update)
def gpu_pass():
    lays, qp, kp = [], [], []
    keys0 = None
    for li in range(NB):
        keys, vals, cen = bench.gen_layer(torch, U, n, d, li, dev)
        if li == 0:
            keys0, vals0 = keys[0].cpu().numpy(), vals[0].cpu().numpy()
        from paper_2505_02922_b200.config import IndexConfig
        ecfg = EngineConfig(cache_fraction=float(os.environ.get("CACHE_FRAC", 0.05)),
                            index=IndexConfig(estimation_fraction=EST_FRAC, retrieval_fraction=RET_FRAC))
        lay = WaveLayer(ecfg, U, G, d, max_prefill=n, max_decode=2048 if UPD else 64, store_dtype=torch.float32 if os.environ.get("STORE") == "f32" else torch.bfloat16,
                        offload=os.environ.get("OFFLOAD") == "1", split=int(os.environ.get("SPLIT", 1)),
                        splits=int(os.environ["SPLITS"]) if "SPLITS" in os.environ else None)
        lay.prefill(keys, vals)
        lays.append(lay)
        qp.append(bench.gen_queries(torch, cen, G, STEPS, 7 + li))
        g = torch.Generator(device=dev); g.manual_seed(11 + li)
        kp.append(torch.randn((STEPS, 2, U, d), device=dev, generator=g).bfloat16().float())
        del keys, vals, cen
    rec = []
    for j in range(STEPS):
        for b in range(NB):
            if UPD:
                lays[b].launch_step(qp[b][j], kp[b][j, 0], kp[b][j, 1])
                for s in lays[b].units:
                    s.total += 1
                    s.n_steady += 1
                if b == 0:
                    rec.append((lays[0].out[0].clone(), lays[0].logden[0].clone(), lays[0].units[0].m,
                                lays[0].cnt.view(U, 4)[0].clone()))
                lays[b].maybe_update()
            else:
                lays[b].launch_step(qp[b][j], kp[b][j, 0], kp[b][j, 1])
                for s in lays[b].units:
                    s.total += 1
                    s.n_steady += 1
                if b == 0:
                    rec.append((lays[0].out[0].clone(), lays[0].logden[0].clone(), lays[0].units[0].m,
                                lays[0].cnt.view(U, 4)[0].clone()))
    torch.cuda.synchronize()
    hist = [(qp[0][j][0].double().cpu().numpy(), kp[0][j, 0][0].cpu().numpy(), kp[0][j, 1][0].cpu().numpy())
            for j in range(STEPS)]
    return rec, hist, keys0, vals0
rec, hist, keys0, vals0 = gpu_pass()
rec2, _, _, _ = gpu_pass()
nd = [j for j in range(STEPS) if not torch.equal(rec[j][0], rec2[j][0])]
print("GPU run-to-run differing steps:", nd[:20])
e0 = O.OracleEngine(blas_threads=8, estimation_fraction=EST_FRAC, retrieval_fraction=RET_FRAC).prefill(keys0, vals0)
orcs = [e0] + [e0.clone() for _ in range(G - 1)]
for j, (q, k, v) in enumerate(hist):
    outs = [orcs[g].decode_step(q[g], k, v, with_recall=False) for g in range(G)]
    o = rec[j][0].double().cpu().numpy()
    errs = [float(np.linalg.norm(o[g] - outs[g][0]) / np.linalg.norm(outs[g][0])) for g in range(G)]
    dl = [abs(float(rec[j][1][g]) - outs[g][1].log_denominator) for g in range(G)]
    flag = "BAD" if max(errs) > 1e-5 else ""
    if UPD and not flag and j % 100 and j < STEPS - 4 and rec[j][2] == rec[max(0, j - 1)][2]:
        continue
    print(f"step {j:3d} rel_l2 {max(errs):.2e} dlog {max(dl):.2e} cnt {rec[j][3].tolist()} "
          f"r/e {[outs[g][1].r for g in range(G)]} m {rec[j][2]} oracle m {orcs[0].m} {flag}")
