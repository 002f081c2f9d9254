"""CPU dry run of the multi-GPU plan for config C5 (R-MAT n=5e7, m=1e9, nnz=2e9; BASELINE.json
configs[4]): generate the graph, partition it with the library's wl_partition (nnz-balanced rows) for
P in {2, 4, 8}, build every rank's halo plan with wl_halo_plan (host only, no GPU) and report the halo
fraction, the halo bytes per SpMM at b = 32 and the device memory per rank that wl_operator_create and a
b = 32 TOAR workspace (k = 30) would allocate.  Output: profiles/r02_c5_dryrun.json."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen as gg  # noqa: E402
from graphgen import configs  # noqa: E402
import paper_2601_11338_b200 as wl  # noqa: E402


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    cfg = configs.get(cfg_name)
    t0 = time.time()
    g = cfg["make"]()
    t_gen = time.time() - t0
    print(f"generated {cfg_name}: n={g.n} nnz={g.nnz} in {t_gen:.0f} s", flush=True)
    b, K = 32, 30
    B = min(32, b * len(cfg["thetas"]))
    out = {"config": cfg_name, "desc": cfg["desc"], "n": g.n, "nnz": g.nnz, "generate_s": round(t_gen, 1),
           "b": b, "krylov_dim": K, "partitions": {}}
    for P in (2, 4, 8):
        bounds = wl.partition(g.row_ptr, P)
        ranks = []
        for r in range(P):
            rb, re = int(bounds[r]), int(bounds[r + 1])
            rp = g.row_ptr[rb:re + 1]
            ci = g.col_idx[rp[0]:rp[-1]]
            t1 = time.time()
            col, halo, cnt = wl.halo_plan(g.n, bounds, r, rp, ci)
            n_loc, nnz_loc, n_halo = re - rb, int(rp[-1] - rp[0]), len(halo)
            n_local_cols = int(np.count_nonzero(col < n_loc))
            # device bytes: CSR (int32 rowptr + col), perm, bins ~ 3 int32 per row; TOAR workspace
            # (K + 5) n-blocks + padded gathered block; halo send/recv at the padded row width
            ldg = (B + 3) // 4 * 4
            csr = 4 * (n_loc + 1) + 4 * nnz_loc + 12 * n_loc
            ws = 8 * (n_loc + 1) * B * (K + 5) + 8 * (n_loc + 1) * ldg
            halo_b = 8 * n_halo * ldg
            ranks.append({"rank": r, "rows": n_loc, "nnz": nnz_loc, "n_halo": n_halo,
                          "halo_over_n_global": n_halo / g.n, "halo_over_n_local": n_halo / max(1, n_loc),
                          "local_nnz_frac": n_local_cols / max(1, nnz_loc),
                          "halo_bytes_per_spmm_b32": halo_b, "device_bytes_csr": csr,
                          "device_bytes_workspace_b32": ws, "device_bytes_halo_buffers": 2 * halo_b,
                          "device_GB_total": round((csr + ws + 2 * halo_b) / 1e9, 2),
                          "plan_s": round(time.time() - t1, 1)})
            print(P, ranks[-1], flush=True)
            del col, halo
        out["partitions"][str(P)] = {
            "bounds": [int(x) for x in bounds],
            "max_halo_over_n_global": max(x["halo_over_n_global"] for x in ranks),
            "max_device_GB": max(x["device_GB_total"] for x in ranks),
            "fits_180GB": max(x["device_GB_total"] for x in ranks) < 170.0,
            "ranks": ranks}
    path = os.path.join(ROOT, "profiles", f"r02_{cfg_name}_dryrun.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
