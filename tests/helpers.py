"""Shared parity helpers: move states between the oracle and the device."""

import numpy as np

import oracle as O
from paper_2404_01931_b200 import SceneSpec


def spec_pair(**kw):
    """(device SceneSpec, oracle Spec) with identical fields."""
    return SceneSpec(**kw), O.Spec(**kw)


def device_arrays(st):
    g, go = st.grid, st.grid_old
    d = {"u": g.u, "v": g.v, "w": g.w, "p": g.p, "label": g.label,
         "uo": go.u, "vo": go.v, "wo": go.w,
         "count": st.hash.count, "offset": st.hash.offset}
    for i, a in enumerate(st.particles.arrays()):
        d[f"part{i}"] = a
    return d


def oracle_arrays(os_):
    d = {"u": os_.u, "v": os_.v, "w": os_.w, "p": os_.p, "label": os_.label,
         "uo": os_.uo, "vo": os_.vo, "wo": os_.wo, "count": os_.count, "offset": os_.offset}
    for i, a in enumerate(os_.parts):
        d[f"part{i}"] = a
    return d


def diff_report(dev, ref, keys=None):
    bad = []
    for k in keys or ref:
        a, b = np.asarray(dev[k]), np.asarray(ref[k])
        if a.shape != b.shape:
            bad.append(f"{k}: shape {a.shape} vs {b.shape}")
        elif a.tobytes() != b.tobytes():
            if a.dtype.kind == "f":
                nz = np.flatnonzero(a != b)
                rel = np.max(np.abs(a - b) / np.maximum(1e-300, np.abs(b)))
                bad.append(f"{k}: {len(nz)} differ (first {nz[:5]}), max rel {rel:.3e}")
            else:
                nz = np.flatnonzero(a != b)
                bad.append(f"{k}: {len(nz)} differ (first {nz[:5]})")
    return bad


def upload(st, os_, dt=None, known=None):
    """Overwrite the device state with an oracle state (plus inter-stage data)."""
    dev = st.device
    dev.set_grid(u=os_.u, v=os_.v, w=os_.w, p=os_.p, label=os_.label)
    dev.set_grid_old(os_.uo, os_.vo, os_.wo)
    dev.set_particles(os_.parts)
    dev.set_hash(os_.offset, os_.count)
    if dt is not None:
        dev.set_dt(dt)
    if known is not None:
        dev.set_known(*known)
