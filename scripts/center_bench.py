"""Timing of NEXT-2 on large sizes: the centring post-pass on a dense n × n G (HBM GB/s) and K̃ (rf_ktilde)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01899_b200 as rf


def main():
    dev = torch.device("cuda:0")
    for n, p in [(65536, 1024), (131072, 512)]:
        g = torch.Generator(device=dev).manual_seed(1)
        X = (torch.randn(n, p, device=dev, generator=g) / p ** 0.5).to(torch.bfloat16)
        V = torch.randn(n, 3, device=dev, generator=g) * 0.03
        A = [[2.0, 0.0, 0.1], [0.0, 2.0, -0.1], [0.1, -0.1, 1.0]]
        Kt = torch.empty(n, n, device=dev)
        ws = torch.empty(rf.rf_ktilde_workspace_size(p, n, "bf16"), dtype=torch.uint8, device=dev)
        rf.rf_profile_enable(True)
        for _ in range(4):
            rf.rf_ktilde(X, V, A, 0.09, 0.37, 0.2, prec="bf16", out="upper", Kt=Kt, ws=ws)
        torch.cuda.synchronize()
        rec = rf.rf_profile_read()
        kt = sorted(ms for nm, ms in rec if nm == "KT_ktilde")[1:]
        prep = sorted(ms for nm, ms in rec if nm == "KT_prep")[1:]
        tri = n * (n + 1) / 2
        print(f"[K̃ n={n} p={p}] GEMM+epilogue {kt[len(kt)//2]:.3f} ms ({p * n * (n + 1.0) / kt[len(kt)//2] / 1e9:.0f} TF/s, "
              f"{4 * tri / kt[len(kt)//2] / 1e6:.0f} GB/s written)  prep {prep[len(prep)//2]:.3f} ms", flush=True)
        # centring post-pass on the upper triangle of Kt (as a stand-in dense symmetric matrix)
        cen_ws = torch.empty(rf.rf_phi_workspace_size(p, n, "bf16"), dtype=torch.uint8, device=dev)
        del ws
        for _ in range(3):
            rf.rf_phi_closed_form(X, act="tanh", tau=1.0, prec="bf16", out="upper_centered", Phi=Kt, ws=cen_ws)
        torch.cuda.synchronize()
        rec = rf.rf_profile_read()
        for nm in ("K5_xtx_eq1", "KC_center_rowsum", "KC_center_apply"):
            t = sorted(ms for k, ms in rec if k == nm)
            if t:
                by = 4 * tri * (2 if nm == "KC_center_apply" else 1)
                print(f"   {nm}: {t[len(t)//2]:.3f} ms ({by / t[len(t)//2] / 1e6:.0f} GB/s of the triangle)", flush=True)
        del Kt, cen_ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
