import sys, os
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1808_04473_b200 import _lib
rng = np.random.default_rng(0)
n, B, U, T = 1, 64, 16, 2
H = ((rng.standard_normal((n, B, U)) + 1j * rng.standard_normal((n, B, U))) / 8).astype(np.complex64)
Y = (rng.standard_normal((n, T, B)) + 1j * rng.standard_normal((n, T, B))).astype(np.complex64)
Hd, Yd = torch.from_numpy(H).cuda(), torch.from_numpy(Y).cuda()
out = torch.zeros((n, 2, U * U + T * U), dtype=torch.complex64, device='cuda')
off, offp = _lib.host_i32([0, 32, 64])
lib = _lib.lib()
lib.dbp_gram_mrc(_lib.ptr(Hd), _lib.ptr(Yd), n, B, U, U, T, 2, offp, 0, _lib.ptr(out), _lib.stream_ptr())
torch.cuda.synchronize()
tile = np.fromfile("gpurun_out/tile_dump.bin", dtype=np.float32)
def elem(f, k):
    qd = k // 4
    off = (f >> 3) * 1024 + (f & 7) * 128 + ((qd ^ (f & 7)) << 4) + (k % 4) * 4
    return tile[off // 4]
YB = 64
for name, rows, ref in (("H_A re u0", [0], H[0, 0:32, 0].real), ("H_B re u0", [32], H[0, 32:64, 0].real),
                        ("Y_A re t0", [YB], Y[0, 0, 0:32].real), ("Y_B re t0", [YB + 2 * T], Y[0, 0, 32:64].real),
                        ("Y_B im t1", [YB + 2 * T + 3], Y[0, 1, 32:64].imag)):
    got = np.array([elem(rows[0], k) for k in range(32)])
    print(name, "max err vs ref %.2e" % np.abs(got - ref).max(), "| vs cluster0 %.2e" % np.abs(got - (Y[0, 0, 0:32].real if 'Y' in name else H[0, 0:32, 0].real)).max())
    print("  got", np.round(got[:6], 3), " ref", np.round(ref[:6], 3))
