import ctypes, sys, os, warnings
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import test_gpu_fit_abi as t
import flowdmd_oracle as orc
import paper_2502_05339_b200 as fd
from conftest import phase_aligned_error
L = t._bind(); ctx = ctypes.c_void_p(); t.chk(L, L.fdmd_ctx_create(0, 2, ctypes.byref(ctx))); abi = (L, ctx)
n, pairs, ell, m = 6000, 5, 3, 61
X, U, true_eigs, Bf = orc.controlled_system(n, pairs, ell, m, seed=7, noise=0.0)
T = m - 1; r_aug, r = 2 * pairs + 2 * ell, 2 * pairs + ell; l_aug, l = r_aug + 10, r + 10
om_aug = np.random.default_rng(5).standard_normal((T, l_aug)); om_out = np.random.default_rng(6).standard_normal((T, l))
M = t.upload(abi, X); sig, lam, red = np.zeros(r_aug), np.zeros(2 * r), np.zeros(2 * r * ell); model = ctypes.c_void_p()
t.chk(L, L.fdmd_dmdc_fit(ctx, M, t._p(U), ell, 1.0, r_aug, l_aug, r, l, 1, t._p(om_aug), t._p(om_out), t._p(sig), t._p(lam), t._p(red), ctypes.byref(model)))
lam = lam[0::2] + 1j * lam[1::2]; red = (red[0::2] + 1j * red[1::2]).reshape(r, ell)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    pm, ctrl = fd.dmdc_fit(fd.SnapshotMatrix(X, 1.0), U, r_aug, r, seed=5, oversample=10, power_iters=1)
print("lam diff", np.abs(np.sort_complex(lam) - np.sort_complex(pm.lam)).max())
phi = t.phi_of(abi, model, n, r)
print("phi vs python", phase_aligned_error(phi, pm.phi), np.abs(phi - pm.phi).max())
print("red vs python", np.abs(red - ctrl.reduced_b[0]).max(), np.abs(ctrl.reduced_b[0]).max())
z = t.encode(abi, model, X[:, 0], r); zp = fd.encode(pm, X[:, 0]).z
print("z0 diff", np.abs(z - zp).max(), np.abs(zp).max())
print("Btil python", pm.provenance["B_tilde"][:3])
# per-column agreement, conditioning, and host rollouts of both models
for k in range(r):
    ip = np.vdot(phi[:, k], pm.phi[:, k]); ph = ip / abs(ip) if abs(ip) > 0 else 1
    print(k, np.round(lam[k], 6), np.round(pm.lam[k], 6), "col err", np.linalg.norm(phi[:, k] * ph - pm.phi[:, k]))
sv = np.linalg.svd(phi, compute_uv=False); svp = np.linalg.svd(pm.phi, compute_uv=False)
print("cond C", sv[0] / sv[-1], "cond py", svp[0] / svp[-1])
zc = np.linalg.lstsq(phi, X[:, 0], rcond=None)[0]
print("encode C vs lstsq", np.abs(z - zc).max() / np.abs(zc).max())
def roll(ph_, l_, rb_, z_):
    w = 0.0
    for k in range(T):
        z_ = l_ * z_ + rb_ @ U[:, k]
        fr = (ph_ @ z_).real
        w = max(w, np.linalg.norm(fr - X[:, k + 1]) / np.linalg.norm(X[:, k + 1]))
    return w
print("rollout C (C red, lstsq z)", roll(phi, lam, red, zc))
rb_ls = np.linalg.lstsq(phi, (X[:, 1:] - (phi @ (lam[:, None] * np.linalg.lstsq(phi, X[:, :-1], rcond=None)[0])).real) @ np.linalg.pinv(U), rcond=None)[0]
print("python rollout", roll(pm.phi, pm.lam, ctrl.reduced_b[0], zp))
