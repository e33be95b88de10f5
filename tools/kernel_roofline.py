"""Per-kernel HBM roofline table from an ncu launch list.

    python tools/kernel_roofline.py gpurun_out/launches_r1e.csv > profiles/r01_kernel_roofline.md

Algorithmic bytes per launch: every input read once, every output written
once (fp64 8 B, int32 4 B, label/mask 1 B), with the 256^3 dam-break sizes
of the captured steps: N particles, C cells, Fc faces per component, R
pressure rows.  ncu times are serialised and cold-cache (--cache-control
all), i.e. pessimistic; the fraction is of the measured 6549 GB/s copy peak.
"""
import collections
import csv
import json
import os
import re
import sys

N = 24.9e6        # mean particle count entering steps 1..4 after warm-up
C = 256 ** 3
FC = 257 * 256 * 256
R = 3.13e6        # pressure rows
PEAK = 6549.4

# kernel -> (bytes per launch, formula text)
BYTES = {
    "k_maxv2": (24 * N, "24N (|v|^2 max)"),
    "k_advect_key": (76 * N + 4 * C, "48N read + 24N pos + 4N key + 4C count"),
    "k_radix_hist": (4 * N, "4N keys per pass"),
    "k_radix_scatter": (16 * N, "8N read + 8N write per pass"),
    "k_gather6": (96 * N, "48N read + 48N write"),
    "k_classify": (6 * C, "count 4C + label 2C"),
    "k_p2g<1>": (32 * N + 4 * C + 17 * FC + C, "pos+vel 32N, offsets 4C, grid+old+known 17Fc, labels C"),
    "k_force_enforce": (16 * FC + C, "16Fc + C"),
    "k_uf_link": (C + 4 * C, "labels + parents"),
    "k_assemble_rows": (8 * 3 * FC / 3 + C + 9 * R, "faces 8F/3 + C + 9R"),
    "k_matvec": (48 * R, "s 8R + diag 8R + nbr 24R + q 8R"),
    "k_matvec_c": (30 * R, "s 8R + meta 2R + dy 4R + dz 8R + q 8R"),
    "k_dot_nodes<LdProd>": (16 * R, "two vectors"),
    "k_dot_nodes<LdLaneDot>": (28 * R, "zL gather 8R + posL 4R + r 8R + z 8R"),
    "k_dot_fused<LdProd>": (16 * R, "two vectors"),
    "k_dot_fused<LdLaneDot>": (28 * R, "zL gather 8R + posL 4R + r 8R + z 8R"),
    "k_wave_prep": (8 * 256 * 32 * 115, "halo refill: tiles x 32 x nsteps doubles"),
    "k_pcg_update": (60 * R, "x,r r/w 32R + s,q 16R + rL 8R + posL 4R"),
    "k_pcg_dir": (24 * R, "z, s read + s write"),
    "k_mic_cl<0, 4, 4, 4, 3, 0>": (24 * R, "src + precon read, dst write"),
    "k_mic_cl<1, 4, 4, 4, 3, 0>": (24 * R, "src + precon read, dst write"),
    "k_gradient": (16 * FC + 8 * C, "face r/w 16Fc + p 8C"),
    "k_extrap_layer": (34 * FC, "grid + grid_old faces r/w + known, one component-layer"),
    "k_g2p": (72 * N + 48 * FC, "particles 72N + grid and grid_old 48Fc"),
    "k_reseed_copy": (100 * N, "96N copy + 4N cell"),
}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("void ", "")
        v = float(r[ix["Metric Value"]])
        u = r[ix["Metric Unit"]]
        v = v / 1000 if u == "ns" else (v if u == "us" else v * 1000)
        agg[name][0] += 1
        agg[name][1] += v
    total = sum(v[1] for v in agg.values())
    print("| kernel | launches | avg µs | share | algorithmic bytes / launch | GB/s | HBM frac |")
    print("|---|---|---|---|---|---|---|")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if us / total < 0.002:
            continue
        avg = us / n
        if k in BYTES:
            b, txt = BYTES[k]
            gbs = b / (avg * 1e-6) / 1e9
            print(f"| `{k}` | {n} | {avg:.1f} | {100 * us / total:.1f}% | {b / 1e6:.0f} MB ({txt}) "
                  f"| {gbs:.0f} | {gbs / PEAK:.1%} |")
        else:
            print(f"| `{k}` | {n} | {avg:.1f} | {100 * us / total:.1f}% | — | — | — |")


if __name__ == "__main__":
    main(sys.argv[1])
