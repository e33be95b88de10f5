"""Digest helpers shared by the golden-fixture tests (see golden/make_golden.py)."""

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()


def load(name):
    return json.load(open(os.path.join(HERE, "golden", name)))


def parse_case(key: str) -> dict:
    out = {}
    # keys are "k=v" joined by ","; gravity tuples contain commas
    parts, cur = [], ""
    for tok in key.split(","):
        cur = tok if not cur else cur + "," + tok
        if cur.count("(") == cur.count(")"):
            parts.append(cur)
            cur = ""
    for p in parts:
        k, v = p.split("=", 1)
        try:
            out[k] = eval(v, {}, {})
        except Exception:
            out[k] = v
    return out


def oracle_digests(os_) -> dict:
    out = {k: digest(getattr(os_, k)) for k in ("u", "v", "w", "p", "label")}
    out.update({"uo": digest(os_.uo), "vo": digest(os_.vo), "wo": digest(os_.wo),
                "count": digest(os_.count.astype(np.int64)),
                "offset": digest(os_.offset.astype(np.int64))})
    for i, a in enumerate(os_.parts):
        out[f"part{i}"] = digest(a)
    out["n"] = int(os_.n)
    return out


def device_digests(st) -> dict:
    g, go = st.grid, st.grid_old
    out = {k: digest(getattr(g, k)) for k in ("u", "v", "w", "p", "label")}
    out.update({"uo": digest(go.u), "vo": digest(go.v), "wo": digest(go.w),
                "count": digest(st.hash.count.astype(np.int64)),
                "offset": digest(st.hash.offset.astype(np.int64))})
    for i, a in enumerate(st.particles.arrays()):
        out[f"part{i}"] = digest(a)
    out["n"] = int(st.particles.count)
    return out


def report_tuple(dt, n, its, res, conv):
    return (float(dt).hex(), int(n), int(its), float(res).hex(), bool(conv))
