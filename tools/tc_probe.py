# layout probe: one-hot channels through dbp_gram_mrc, print where G's mass lands
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1808_04473_b200 import _lib
B, U, T = 32, 16, 2
lib = _lib.lib()
def run(H, Y):
    n = H.shape[0]
    Hd, Yd = torch.from_numpy(H).cuda(), torch.from_numpy(Y).cuda()
    out = torch.zeros((n, 1, U * U + T * U), dtype=torch.complex64, device='cuda')
    off, offp = _lib.host_i32([0, B])
    _lib.check(lib.dbp_gram_mrc(_lib.ptr(Hd), _lib.ptr(Yd), n, B, U, U, T, 1, offp, 0, _lib.ptr(out), _lib.stream_ptr()))
    return out.cpu().numpy()[:, 0]
for (k0, u0) in [(0, 0), (0, 1), (1, 0), (0, 2), (3, 5), (9, 0), (8, 4)]:
    H = np.zeros((1, B, U), np.complex64); H[0, k0, u0] = 1.0
    Y = np.zeros((1, T, B), np.complex64)
    o = run(H, Y)[0]
    G = o[:U * U].reshape(U, U)
    nz = [(i, j, np.round(G[i, j], 3)) for i, j in zip(*np.nonzero(np.abs(G) > 1e-6))]
    print("H one-hot", (k0, u0), "G nz:", nz[:8])
rng = np.random.default_rng(0)
H = ((rng.standard_normal((1, B, U)) + 1j * rng.standard_normal((1, B, U))) / 8).astype(np.complex64)
Y = np.zeros((1, T, B), np.complex64)
o = run(H, Y)[0]
G = o[:U * U].reshape(U, U); Gr = H[0].conj().T @ H[0]
print("random G err", np.abs(G - Gr).max(), "scale", np.abs(Gr).max())
for (t0, k0) in [(0, 0), (1, 0), (0, 1), (0, 5)]:
    H = np.zeros((1, B, U), np.complex64); H[0, :, 0] = 1.0
    Y = np.zeros((1, T, B), np.complex64); Y[0, t0, k0] = 1.0
    o = run(H, Y)[0]
    Z = o[U * U:].reshape(T, U)
    nz = [(i, j, np.round(Z[i, j], 3)) for i, j in zip(*np.nonzero(np.abs(Z) > 1e-6))]
    print("Y one-hot", (t0, k0), "Z nz:", nz[:8])
