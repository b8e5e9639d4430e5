"""CPU check of the algebra behind the tensor-core K1 (paper_2202_07848_b200/csrc/k_hash_mma.cu):
FNV-1a-64 over a page (sim.hpp:55-65) equals H0 P^n + P^-(4096-n) (S + l_4096 - 0x25 P^4096),
where S = sum_j D_j << 8j and D = the u8 x u8 -> s32 product of the two byte streams the CUDA
cores produce (two pages per 32-bit register, 16-bit lanes) with the byte limbs of the weights
P^(4096-t) / -P^(4096-t). This restates the kernel's data flow step by step (same packing, same
batch layout of the B operand) in Python, against the reference FNV-1a (oracle.digest_of_bytes)."""
import numpy as np
import pytest

import oracle as O

M64 = (1 << 64) - 1
P = 0x100000001B3
H0 = 0xCBF29CE484222325
BSTEPS = 32  # byte-steps per MMA batch


def weights():
    """B operand per batch: 16 rows (limbs of page a, limbs of page b) x 128 K-bytes
    (u words | l words), as make_btab() lays it out (before the SW128 swizzle)."""
    bt = np.zeros((4096 // BSTEPS, 16, 128), np.int64)
    for bi in range(4096 // BSTEPS):
        t0 = BSTEPS * bi
        for m in range(BSTEPS // 2):
            for j in range(4):
                pg, dt = j >> 1, j & 1
                wu = pow(P, 4096 - (t0 + 2 * m + dt), 1 << 64)
                wl = (-pow(P, 4096 - (t0 + 2 * m + 1 + dt), 1 << 64)) & M64
                for n in range(8):
                    bt[bi, 8 * pg + n, 4 * m + j] = (wu >> (8 * n)) & 255
                    bt[bi, 8 * pg + n, 2 * BSTEPS + 4 * m + j] = (wl >> (8 * n)) & 255
    return bt


@pytest.fixture(scope="module")
def btab():
    return weights()


def kernel_model(pa, pb, na, nb, bt):
    """Digests of two pages (byte arrays of 4096, zero past n) the way one thread + the MMA
    compute them."""
    L = 0x00250025  # l_0 = 0x25 in both 16-bit lanes
    D = np.zeros(16, np.int64)
    for bi in range(4096 // BSTEPS):
        upk, lpk = [], []
        prev_u = prev_l = 0
        for k in range(BSTEPS):
            t = BSTEPS * bi + k
            x = int(pa[t]) | (int(pb[t]) << 16)          # PRMT: byte t of both pages
            u = (L ^ x) & 0x00FF00FF                     # LOP3
            Lp = L
            L = (u * 179) & 0xFFFFFFFF                   # IMAD: low bytes = next l
            if k & 1:
                upk.append((prev_u + (u << 8)) & 0xFFFFFFFF)   # [u_a,k u_a,k+1 u_b,k u_b,k+1]
                # PRMT(L_k, L_k+1, 0x6240) = [l_a,k+1 l_a,k+2 l_b,k+1 l_b,k+2]
                lpk.append((Lp & 0xFF) | ((L & 0xFF) << 8) | (((Lp >> 16) & 0xFF) << 16)
                           | (((L >> 16) & 0xFF) << 24))
            else:
                prev_u = u
        a_row = np.frombuffer(np.array(upk + lpk, np.uint32).tobytes(), np.uint8).astype(np.int64)
        D += bt[bi] @ a_row                              # tcgen05.mma kind::i8, s32 accumulate
    assert D.max() < 2 ** 31
    out = []
    k0 = (0x25 * pow(P, 4096, 1 << 64)) & M64
    inv = pow(P, -1, 1 << 64)
    for pg, n, sh in ((0, na, 0), (1, nb, 16)):
        S = sum(int(D[8 * pg + j]) << (8 * j) for j in range(8)) & M64
        ln = (L >> sh) & 0xFF
        hp = (H0 * pow(P, n, 1 << 64)) & M64
        ip = pow(inv, 4096 - n, 1 << 64)
        out.append((hp + ip * ((S + ln - k0) & M64)) & M64)
    return out


@pytest.mark.parametrize("na,nb", [(4096, 4096), (256, 4096), (3840, 1024), (4096, 768)])
def test_decomposition_matches_fnv(btab, na, nb):
    rng = np.random.default_rng(na * 7 + nb)
    pa = np.zeros(4096, np.uint8)
    pb = np.zeros(4096, np.uint8)
    pa[:na] = rng.integers(0, 256, na, dtype=np.uint8)
    pb[:nb] = rng.integers(0, 256, nb, dtype=np.uint8)
    ha, hb = kernel_model(pa, pb, na, nb, btab)
    assert ha == O.digest_of_bytes(pa[:na].tobytes())
    assert hb == O.digest_of_bytes(pb[:nb].tobytes())
