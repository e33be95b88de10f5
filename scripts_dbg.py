import os, sys
import numpy as np
sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import paper_2404_01931_b200 as P, oracle as O
for res in (12, 20, 40):
    spec = P.SceneSpec(name="dam-break", res=res, max_iters=0)
    st = P.make_scene(spec, 3)
    ospec = O.Spec(name="dam-break", res=res)
    os_ = O.make_scene(ospec, 3)
    cap = {}
    O.step(os_, ospec, hook=lambda n, s, e: cap.update(e) if n == "project" else None)
    rep = P.run_stages(st, spec, "dt_compute", "project")
    sys_ = cap["system"]; n = sys_.nrows
    pc_ref = np.empty(n)
    O.lib().orc_mic0_build(n, O._p(sys_.diag), O._p(sys_.nbr_rows.reshape(-1), O._i64), sys_.scale, 0.97, 0.25, O._p(pc_ref))
    pc = st.device.debug_buffer("precon", n)
    bad = np.flatnonzero(pc != pc_ref)
    cells = sys_.cells
    print(res, "rows", n, rep.nrows, "precon mismatches", len(bad), "first cells", [(c % res, c // res % res, c // res // res) for c in cells[bad[:8]]])
    q_ref = np.zeros(n); z_ref = np.empty(n)
    O.lib().orc_mic0_apply(n, O._p(pc_ref), O._p(sys_.nbr_rows.reshape(-1), O._i64), O._p(sys_.rhs), sys_.scale, O._p(q_ref), O._p(z_ref))
    tq = st.device.debug_buffer("tq", n); z = st.device.debug_buffer("z", n)
    bq = np.flatnonzero(tq != q_ref); bz = np.flatnonzero(z != z_ref)
    print("   fwd mismatches", len(bq), [(c % res, c // res % res, c // res // res) for c in cells[bq[:6]]],
          "bwd mismatches", len(bz), [(c % res, c // res % res, c // res // res) for c in cells[bz[:6]]])
    if len(bz):
        k = bz[0]; print("   z", z[k], z_ref[k], "nbr", sys_.nbr_rows[k])
