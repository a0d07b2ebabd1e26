"""CPU model of the tensor-core fused pass (engine/fused.cuh,
fused_pass_mma_kernel) for one warp and one register group: the lane /
register bit schedule (planner, fused.cpp), the shuffle exchanges
(mma_exchange), the m8n8k4 fragment layouts of mma_apply (A: row = team t,
col = lane j; B: [k = j][n = t]; D: [t][2j, 2j+1]) and the load / store
addressing — restated statement by statement with numpy lanes and checked
against applying the same 4x4 blocks to the hexads directly."""
import numpy as np


def schedule(blocks):
    """fused.cpp: lane bits start on the first block's bits; before each
    block a lane bit it does not use is swapped with a register bit it uses."""
    lane = [blocks[0][0], blocks[0][1]]
    reg = [i for i in range(4) if i not in lane]
    init = lane + reg
    out = []
    for gb0, gb1 in blocks:
        xs = []
        for p in (0, 1):
            if lane[p] in (gb0, gb1):
                continue
            q = 0 if reg[0] in (gb0, gb1) else 1
            lane[p], reg[q] = reg[q], lane[p]
            xs.append((p, q))
        out.append((xs, lane[0] != gb0))
    return init, out, lane + reg


def mma(A, B, C):
    """m8n8k4 over a warp: A[t][j] (lane 4t+j), B[j][t] (lane 4t+j), C/D[t][2j:2j+2]."""
    Am = np.array(A).reshape(8, 4)
    Bm = np.array(B).reshape(8, 4).T  # B[k][n] from lane (n, k)
    Dm = Am @ Bm + np.array(C).reshape(8, 8)
    return Dm.reshape(32, 2)


def test_mma_group_model():
    rng = np.random.default_rng(5)
    for trial in range(200):
        nblk = int(rng.integers(1, 5))
        blocks = []
        for _ in range(nblk):
            a, b = sorted(rng.choice(4, 2, replace=False))
            blocks.append((int(a), int(b)))
        mats = [rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)) for _ in blocks]
        hexads = rng.normal(size=(32, 16)) + 1j * rng.normal(size=(32, 16))  # warp's 32 hexads
        # reference: apply each block to each hexad (matrix bit 0 <-> gb0)
        want = hexads.copy()
        for (g0, g1), M in zip(blocks, mats):
            for h in range(32):
                for rest in range(16):
                    if rest & ((1 << g0) | (1 << g1)):
                        continue
                    idx = [rest | ((c & 1) << g0) | ((c >> 1) << g1) for c in range(4)]
                    want[h, idx] = M @ want[h, idx]
        init, sched, fin = schedule(blocks)
        # load: lane (t, j) register r = hh*4 + rb holds element (j bits -> init[0:2], rb bits -> init[2:4])
        def elem(lay, j, rb):
            return ((j & 1) << lay[0]) | ((j >> 1) << lay[1]) | ((rb & 1) << lay[2]) | ((rb >> 1) << lay[3])
        a = np.zeros((32, 16), complex)
        for lane in range(32):
            t, j = lane >> 2, lane & 3
            for r in range(16):
                a[lane, r] = hexads[t * 4 + (r >> 2), elem(init, j, r & 3)]
        for ((g0, g1), M), (xs, perm) in zip(zip(blocks, mats), sched):
            for p, q in xs:  # mma_exchange<P, Q>
                new = a.copy()
                for lane in range(32):
                    b = (lane & 3) >> p & 1
                    for r0 in range(16):
                        if r0 & (1 << q):
                            continue
                        r1 = r0 | (1 << q)
                        partner = lane ^ (1 << p)
                        pb = (partner & 3) >> p & 1
                        psend = a[partner, r0] if pb else a[partner, r1]
                        if b:
                            new[lane, r0] = psend
                        else:
                            new[lane, r1] = psend
                a = new
            # mma_apply
            sw = (lambda x: ((x & 1) << 1) | (x >> 1)) if perm else (lambda x: x)
            b1 = np.zeros(32)
            b2 = np.zeros(32)
            for lane in range(32):
                t, j = lane >> 2, lane & 3
                m = M[sw(t >> 1), sw(j)]
                b1[lane] = m.imag if t & 1 else m.real
                b2[lane] = m.real if t & 1 else -m.imag
            for r in range(16):
                d = mma(a[:, r].real, b1, np.zeros((32, 2)))
                d = mma(a[:, r].imag, b2, d)
                a[:, r] = d[:, 0] + 1j * d[:, 1]
        got = np.zeros_like(hexads)
        for lane in range(32):
            t, j = lane >> 2, lane & 3
            for r in range(16):
                got[t * 4 + (r >> 2), elem(fin, j, r & 3)] = a[lane, r]
        assert np.allclose(got, want, atol=1e-12), (trial, blocks)
