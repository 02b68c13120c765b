"""Helpers to load the committed tierkv golden fixtures (tests/golden/)."""
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bf16_round(x):
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def manifest():
    with open(os.path.join(GOLDEN, "MANIFEST.json")) as f:
        return json.load(f)


def rank_cases():
    z = load("rank.npz")
    cases = {}
    for key in z.files:
        case, field = key.split("__")
        cases.setdefault(case, {})[field] = z[key]
    out = []
    for name, c in sorted(cases.items()):
        cr = np.random.default_rng(int(c["seed"]))
        m, d = int(c["m"]), int(c["d"])
        C = cr.standard_normal((m, d)) * 0.25 + cr.standard_normal((1, d))
        Q = bf16_round(cr.standard_normal((8, d)).astype(np.float32)).astype(np.float64)
        assert sha(C) == str(c["C_sha"]), "numpy generator drifted; regenerate goldens"
        c.update(C=C, Q=Q)
        out.append((name, c))
    return out


def topk_case():
    z = load("topk.npz")
    kr = np.random.default_rng(int(z["keys_seed"]))
    keys = bf16_round(kr.standard_normal((60000, 128)).astype(np.float32))
    assert sha(keys) == str(z["keys_sha"])
    return keys, z


def engine_case(name):
    z = load(name + ".npz")
    cfg = json.loads(str(z["config"]))
    return z, cfg


def split(flat, lens):
    out, p = [], 0
    for n in lens:
        out.append(flat[p:p + n])
        p += n
    return out
