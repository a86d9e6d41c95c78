"""Seeded synthetic snapshot streams shaped like the paper's workloads.

Stand-ins for the datasets the paper uses but that are not available here
(JHU channel flow P:725, ignition P:726, NSTX GPI P:727); see DESIGN.md
section 5 for the recipes and which BASELINE.json config each one serves.

This module only produces input matrices (and config constants).  It holds
none of the method's arithmetic, so both the oracle and the CUDA path can
consume its output.  Parity sizes are generated on the host with numpy (the
GPU path uploads the same bytes); throughput sizes are generated on the
device with torch outside any timed region.
"""

from dataclasses import dataclass
import math

import numpy as np


# --------------------------------------------------------------------------- configs

@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    b: int
    k: int
    ell: int
    split: tuple
    dtype: str          # "f64" | "f32"
    lam: float          # >= 0 fixed (C1: computed by the harness), -1 paper surrogate
    data_seed: int


def hutch_split(ell):
    """floor(l/6), floor(l/3), rest (reading R11)."""
    a, b = ell // 6, ell // 3
    return (a, b, ell - a - b)


C1 = Config("C1", 4096, 512, 16, 20, 48, (16, 16, 16), "f64", math.nan, 1001)
C2 = Config("C2", 64 * 80, 20000, 64, 100, 256, hutch_split(256), "f32", -1.0, 1002)
C3 = Config("C3", 3 * 192 * 129 * 192, 1000, 32, 200, 512, hutch_split(512), "f64", -1.0, 1003)
C3R = Config("C3r", 3 * 48 * 33 * 48, 1000, 32, 200, 512, hutch_split(512), "f64", -1.0, 1003)
C4 = Config("C4", 10 * 1024 * 1024, 2000, 32, 300, 640, hutch_split(640), "f64", -1.0, 1004)
C4R = Config("C4r", 10 * 32 * 32, 2000, 32, 300, 640, hutch_split(640), "f64", -1.0, 1004)
C5 = Config("C5", 1 << 27, 4096, 64, 400, 1024, hutch_split(1024), "f32", -1.0, 1005)
C5R = Config("C5r", 1 << 18, 4096, 64, 400, 1024, hutch_split(1024), "f32", -1.0, 1005)
CONFIGS = {c.name: c for c in (C1, C2, C3, C3R, C4, C4R, C5, C5R)}


# --------------------------------------------------------------------------- C1

def c1_matrix(seed=1001, m=4096, n=512, rank=10, noise=1e-6):
    """BASELINE config 0: A = U diag(sigma) V^T + 1e-6 N(0,1), sigma_i = 10^(-i/3).

    U, V: seeded random orthonormal (QR of Gaussian, sign-fixed so diag(R) > 0).
    """
    rng = np.random.default_rng(seed)
    U, R = np.linalg.qr(rng.standard_normal((m, rank)))
    U = U * np.sign(np.diag(R))
    V, R = np.linalg.qr(rng.standard_normal((n, rank)))
    V = V * np.sign(np.diag(R))
    sig = 10.0 ** (-np.arange(1, rank + 1) / 3.0)
    return (U * sig) @ V.T + noise * rng.standard_normal((m, n))


def low_rank_matrix(seed, m, n, rank, noise=0.0, decay=None):
    """Generic exactly-rank-r (+ optional noise) matrix for pins and edge cases."""
    rng = np.random.default_rng(seed)
    U = rng.standard_normal((m, rank))
    V = rng.standard_normal((n, rank))
    s = np.ones(rank) if decay is None else decay ** np.arange(rank)
    A = (U * s) @ V.T
    if noise:
        A = A + noise * rng.standard_normal((m, n))
    return A


# --------------------------------------------------------------------------- C2

class ImageStream:
    """BASELINE config 1 (NSTX GPI stand-in): 64x80 frames, fp32, pixel i = y*80 + x.

    Frame t = (B(x,y,t) + sum_{j<40} a_j exp(-|(x,y) - c_j(t)|^2 / (2 w_j^2))) (1 + 0.01 N(0,1)),
    a_j = exp(0.5 g_j) (log-normal), w_j ~ U[2,6] px, c_j(t) = c_j(0) + v_j t,
    v_j ~ N(0, 0.05^2) px/frame, periodic wrap; B = 0.2 + 0.1 sin(2 pi t/5000 + phi) + 0.05 x/80.
    """

    H, W, NBLOB = 64, 80, 40

    def __init__(self, seed=1002):
        rng = np.random.default_rng(seed)
        self.seed = seed
        self.amp = np.exp(0.5 * rng.standard_normal(self.NBLOB))
        self.width = rng.uniform(2.0, 6.0, self.NBLOB)
        self.c0 = np.stack([rng.uniform(0, self.W, self.NBLOB), rng.uniform(0, self.H, self.NBLOB)], 1)
        self.vel = 0.05 * rng.standard_normal((self.NBLOB, 2))
        self.phi = rng.uniform(0, 2 * np.pi)

    def block(self, t0, t1, dtype=np.float32):
        y, x = np.mgrid[0:self.H, 0:self.W]
        x = x.reshape(-1).astype(np.float64)
        y = y.reshape(-1).astype(np.float64)
        out = np.empty((self.H * self.W, t1 - t0), dtype=np.float64)
        for jj, t in enumerate(range(t0, t1)):
            c = self.c0 + self.vel * t
            cx = np.mod(c[:, 0], self.W)[:, None]
            cy = np.mod(c[:, 1], self.H)[:, None]
            dx = np.mod(x[None, :] - cx + self.W / 2, self.W) - self.W / 2
            dy = np.mod(y[None, :] - cy + self.H / 2, self.H) - self.H / 2
            blobs = self.amp[:, None] * np.exp(-(dx * dx + dy * dy) / (2 * self.width[:, None] ** 2))
            bg = 0.2 + 0.1 * np.sin(2 * np.pi * t / 5000.0 + self.phi) + 0.05 * x / 80.0
            noise = np.random.default_rng([self.seed, t]).standard_normal(x.size)
            out[:, jj] = (bg + blobs.sum(0)) * (1.0 + 0.01 * noise)
        return out.astype(dtype)


# --------------------------------------------------------------------------- C4

class ReactingFront:
    """BASELINE config 3 (ignition stand-in), fp64: nf = 10 fields (temperature + 9 species)
    on an N x N grid of the unit square, field f at rows [f N^2, (f+1) N^2), node (i, j) at
    f N^2 + i N + j (reading Q17's layout).  Snapshot t: a tanh front of width 0.01 around a seeded
    centre, radius r0 + v t with 20 sinusoidal wrinkle modes (amplitude ~1e-2, travelling),
        T(x, t) = (1 + tanh((R(theta, t) - |x - c|) / 0.01)) / 2,
    species f = s_f (T shifted by a seeded offset of the front, or its complement), s_f log-spaced
    on [1e-6, 1] - the fields span six decades, as in the paper's ignition data.
    """

    def __init__(self, N=1024, nf=10, n=2000, seed=1004):
        rng = np.random.default_rng(seed)
        self.N, self.nf, self.n, self.seed = N, nf, n, seed
        self.m = nf * N * N
        self.c = 0.5 + 0.05 * rng.standard_normal(2)
        self.r0 = 0.05
        self.v = rng.uniform(0.15, 0.2) / n            # radius grows by ~0.15-0.2 over the stream
        self.amp = 0.01 * rng.uniform(0.2, 1.0, 20) / np.arange(1, 21) ** 0.5
        self.mode = np.arange(1, 21) + rng.integers(0, 3, 20)
        self.phi = rng.uniform(0, 2 * np.pi, 20)
        self.omega = rng.uniform(-0.01, 0.01, 20)
        self.scale = np.logspace(0, -6, nf)             # temperature O(1) ... species down to 1e-6
        self.shift = np.concatenate([[0.0], 0.01 * rng.standard_normal(nf - 1)])
        self.sign = np.concatenate([[1.0], rng.choice([-1.0, 1.0], nf - 1)])

    def block(self, t0, t1, row_begin=0, row_end=None):
        N = self.N
        row_end = self.m if row_end is None else row_end
        i, j = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
        x, y = (i / (N - 1)).ravel() - self.c[0], (j / (N - 1)).ravel() - self.c[1]
        r, th = np.hypot(x, y), np.arctan2(y, x)
        out = np.empty((self.m, t1 - t0))
        for jj, t in enumerate(range(t0, t1)):
            R = (self.r0 + self.v * t) * (1.0 + np.sum(self.amp[:, None] * np.sin(
                self.mode[:, None] * th[None, :] + self.phi[:, None] + self.omega[:, None] * t), axis=0))
            for f in range(self.nf):
                T = 0.5 * (1.0 + np.tanh((R + self.shift[f] - r) / 0.01))
                if self.sign[f] < 0:
                    T = 1.0 - T
                out[f * N * N:(f + 1) * N * N, jj] = self.scale[f] * T
        return out[row_begin:row_end]


# --------------------------------------------------------------------------- C3

class ChannelFlow:
    """BASELINE config 2 (JHU channel-flow stand-in), fp64.

    u, v, w on x: Nx periodic [0, 8 pi), y: Ny Chebyshev-Gauss-Lobatto cos(pi j/(Ny-1)),
    z: Nz periodic [0, 3 pi).  Row = ((c*Nz + z)*Ny + y)*Nx + x.
    u_c = [c == 0](1 - y^2) + sum_q A_q Re[e_{c,q} exp(i(alpha_q x/4 + 2 beta_q z/3 - omega_q t + phi_q))]
          T_{n_q}(y) (1 - y^2) + 1e-4 N(0, 1),
    300 distinct (alpha, beta, n_q) in [0,31]^2 x [0,16] minus alpha = beta = 0,
    A_q = A0 kappa_q^(-5/3), kappa_q = |(alpha, beta, n_q)|, omega_q = c_q |(alpha/4, 2 beta/3)|,
    c_q ~ U[0.5, 0.9], A0 set for fluctuation RMS ~0.1.
    """

    NMODE = 300

    def __init__(self, nx=192, ny=129, nz=192, seed=1003, noise=1e-4):
        self.nx, self.ny, self.nz = nx, ny, nz
        self.m = 3 * nx * ny * nz
        self.seed, self.noise = seed, noise
        rng = np.random.default_rng(seed)
        cand = [(a, b, n) for a in range(32) for b in range(32) for n in range(17) if (a, b) != (0, 0)]
        pick = rng.choice(len(cand), self.NMODE, replace=False)
        modes = np.array([cand[i] for i in pick], dtype=np.float64)
        self.alpha, self.beta, self.nq = modes[:, 0], modes[:, 1], modes[:, 2].astype(int)
        kappa = np.sqrt(self.alpha ** 2 + self.beta ** 2 + self.nq ** 2)
        self.phase = rng.uniform(0, 2 * np.pi, self.NMODE)
        speed = rng.uniform(0.5, 0.9, self.NMODE)
        self.omega = speed * np.sqrt((self.alpha / 4) ** 2 + (2 * self.beta / 3) ** 2)
        e = rng.standard_normal((3, self.NMODE)) + 1j * rng.standard_normal((3, self.NMODE))
        self.evec = e / np.linalg.norm(e, axis=0)
        self.y = np.cos(np.pi * np.arange(ny) / (ny - 1))
        self.x = 8 * np.pi * np.arange(nx) / nx
        self.z = 3 * np.pi * np.arange(nz) / nz
        # g_q(y) = T_n(y)(1 - y^2)
        self.g = np.cos(self.nq[None, :] * np.arccos(np.clip(self.y, -1, 1))[:, None]) * (1 - self.y ** 2)[:, None]
        w = kappa ** (-5.0 / 3.0)
        var = np.sum(w ** 2 * 0.5 * np.mean(self.g ** 2, axis=0) / 3.0)
        self.amp = 0.1 * w / math.sqrt(var)

    def _coeff(self, t0, t1):
        t = np.arange(t0, t1, dtype=np.float64)
        ph = np.exp(1j * (self.phase[:, None] - self.omega[:, None] * t[None, :]))   # [Q, T]
        return self.amp[None, :, None] * self.evec[:, :, None] * ph[None]            # [3, Q, T]

    def block(self, t0, t1):
        """Host (numpy) block, m x (t1 - t0) fp64."""
        a = self._coeff(t0, t1)
        ex = np.exp(1j * self.alpha[None, :] * self.x[:, None] / 4)                 # [Nx, Q]
        ez = np.exp(1j * 2 * self.beta[None, :] * self.z[:, None] / 3)              # [Nz, Q]
        nt = t1 - t0
        out = np.empty((3, self.nz, self.ny, self.nx, nt))
        for zi in range(self.nz):
            F = (ez[zi][None, None, :] * self.g[:, None, :] * ex[None, :, :]).reshape(-1, self.NMODE)
            for c in range(3):
                out[c, zi] = (F @ a[c]).real.reshape(self.ny, self.nx, nt)
        out[0] += (1 - self.y ** 2)[None, :, None, None]
        out = out.reshape(self.m, nt)
        for j, t in enumerate(range(t0, t1)):
            out[:, j] += self.noise * np.random.default_rng([self.seed, t]).standard_normal(self.m)
        return out

    def block_torch(self, t0, t1, device, out=None, row_begin=0, row_end=None):
        """Device (torch) block, rows [row_begin, row_end), column-major (rows contiguous).

        Returns a tensor of shape (t1 - t0, m_loc) whose row j is snapshot t0 + j, i.e.
        the column-major m_loc x ncols matrix with leading dimension m_loc.
        """
        import torch
        row_end = self.m if row_end is None else row_end
        nt = t1 - t0
        m_loc = row_end - row_begin
        if out is None:
            out = torch.empty((nt, m_loc), dtype=torch.float64, device=device)
        a = torch.from_numpy(self._coeff(t0, t1)).to(device)                         # [3, Q, T]
        ex = torch.from_numpy(np.exp(1j * self.alpha[None, :] * self.x[:, None] / 4)).to(device)
        ez = torch.from_numpy(np.exp(1j * 2 * self.beta[None, :] * self.z[:, None] / 3)).to(device)
        g = torch.from_numpy(self.g).to(device)
        mean_u = torch.from_numpy(1 - self.y ** 2).to(device)
        plane = self.ny * self.nx
        # iterate over (c, z) planes intersecting the row range
        p0, p1 = row_begin // plane, (row_end + plane - 1) // plane
        for pidx in range(p0, p1):
            c, zi = divmod(pidx, self.nz)
            F = (ez[zi][None, None, :] * g[:, None, :].to(ez.dtype) * ex[None, :, :]).reshape(plane, self.NMODE)
            blk = (F @ a[c]).real                                                      # [plane, T]
            if c == 0:
                blk = blk + mean_u.repeat_interleave(self.nx)[:, None]
            r0, r1 = pidx * plane, (pidx + 1) * plane
            s0, s1 = max(r0, row_begin), min(r1, row_end)
            out[:, s0 - row_begin:s1 - row_begin] = blk[s0 - r0:s1 - r0].T
        gen = torch.Generator(device=device)
        for j, t in enumerate(range(t0, t1)):
            gen.manual_seed((self.seed * 1_000_003 + t) & 0x7FFFFFFFFFFFFFFF)
            out[j].add_(torch.randn(m_loc, generator=gen, device=device, dtype=torch.float64), alpha=self.noise)
        return out


# --------------------------------------------------------------------------- C5

class LowRankStream:
    """BASELINE config 4 (scaling sweep): X = U diag(sigma) V^T + 1e-5 N(0, 1), rank 500 with
    sigma_i = i^-1.5, U (m x 500) and V (n x 500) with unnormalized N(0, 1) entries (SURVEY Q20:
    signal entry variance ~zeta(3) ~ 1.2, noise 1e-5 relative), fp32, m = 2^27 rows (Q16) split
    into contiguous slabs; C5r keeps n, b, k, l and reduces m to 2^18 for parity.

    Host blocks (numpy, parity sizes): U rows from PCG64 keyed on (seed, 1, row chunk of 2^16), V
    from (seed, 2), noise of column t from (seed, 3, t).  Device blocks (torch, throughput sizes)
    follow the same formula with torch's generator (U in row chunks keyed on (seed, chunk)), so
    they have the same structure but not the host's values.
    """

    RANK = 500
    CHUNK = 1 << 16

    def __init__(self, m=1 << 27, n=4096, seed=1005, noise=1e-5):
        self.m, self.n, self.seed, self.noise = m, n, seed, noise
        self.sigma = np.arange(1, self.RANK + 1, dtype=np.float64) ** -1.5
        self.V = np.random.default_rng([seed, 2]).standard_normal((n, self.RANK))

    def _u_rows(self, r0, r1):
        out = np.empty((r1 - r0, self.RANK))
        c0, c1 = r0 // self.CHUNK, (r1 + self.CHUNK - 1) // self.CHUNK
        for c in range(c0, c1):
            u = np.random.default_rng([self.seed, 1, c]).standard_normal((self.CHUNK, self.RANK))
            a, b = max(r0, c * self.CHUNK), min(r1, (c + 1) * self.CHUNK)
            out[a - r0:b - r0] = u[a - c * self.CHUNK:b - c * self.CHUNK]
        return out

    def block(self, t0, t1, row_begin=0, row_end=None):
        """Host (numpy) block, rows [row_begin, row_end) x snapshots [t0, t1), fp32."""
        row_end = self.m if row_end is None else row_end
        U = self._u_rows(row_begin, row_end)
        X = (U * self.sigma) @ self.V[t0:t1].T
        for j, t in enumerate(range(t0, t1)):
            nz = np.random.default_rng([self.seed, 3, t]).standard_normal(self.m)
            X[:, j] += self.noise * nz[row_begin:row_end]
        return X.astype(np.float32)

    def block_torch(self, t0, t1, device, row_begin=0, row_end=None, chunk=1 << 21):
        """Device (torch) block (t1 - t0, m_loc) fp32 (row j = snapshot t0 + j, rows contiguous), as
        a GEMM over row chunks with U generated on the device; outside any timed region."""
        import torch
        row_end = self.m if row_end is None else row_end
        m_loc = row_end - row_begin
        out = torch.empty((t1 - t0, m_loc), dtype=torch.float32, device=device)
        W = torch.from_numpy(self.sigma[:, None] * self.V[t0:t1].T).to(device=device, dtype=torch.float32)  # [R, T]
        gen = torch.Generator(device=device)
        for r in range(row_begin, row_end, chunk):
            r1 = min(row_end, r + chunk)
            gen.manual_seed((self.seed * 1_000_003 + r // chunk) & 0x7FFFFFFFFFFFFFFF)
            U = torch.randn((r1 - r, self.RANK), generator=gen, device=device, dtype=torch.float32)
            out[:, r - row_begin:r1 - row_begin] = (U @ W).T
        for j, t in enumerate(range(t0, t1)):
            gen.manual_seed((self.seed * 7_000_003 + t) & 0x7FFFFFFFFFFFFFFF)
            out[j].add_(torch.randn(m_loc, generator=gen, device=device, dtype=torch.float32), alpha=self.noise)
        return out
