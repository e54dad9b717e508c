"""Solve time of each preconditioner alone on an SM share, per fused-CG
kernel choice (VOXSCHUR_CG 1 = k_cg1, 2 = k_pcg, unset = size rule).
usage: python tools/share_probe.py [C1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)
grid = configs.make_geometry(key)
s = vx.assemble(grid, 0)
for prec, shares in (("uzawa", (40, 46, 52, 60, 74)), ("simple", (90, 96, 101, 108, 148))):
    cfg = vx.SchurConfig(prec=prec, **TOL)
    for sms in shares:
        out = []
        for cg in ("", "1", "2"):
            if cg:
                os.environ["VOXSCHUR_CG"] = cg
            else:
                os.environ.pop("VOXSCHUR_CG", None)
            s.limit_sms(sms)
            vx.solve_schur(s, cfg, return_fields=False)
            r = vx.solve_schur(s, cfg, return_fields=False)
            st = vx.last_kernel_stats(s)
            out.append(f"CG={cg or 'auto'}:{r.device_ms:7.1f} ms ({st['velocity_cg']['kernel']})")
        print(f"{prec:6s} sms {sms:3d}: " + "  ".join(out), flush=True)
