"""Seeded synthetic workloads shared by the tests, bench.py and smoke().

This module only DRAWS inputs (region lengths, CSR offsets, element values)
and names the workload configurations of BASELINE.json; it contains none of
the method's arithmetic (no filtering, no enumeration, no aggregation).  Both
the oracle and the CUDA path consume the very same arrays produced here.

Workload recipes:
  D1 tiny   : R = 1000, lengths U{1..64}, int32 full range, 2 x HASH_LT(T=192), SUM_I64
  D2 sweep  : region lengths fixed L or U{0..2L}, L in {1,4,32,256,4096};
              int32 full range, 3 x HASH_LT(T=192), SUM_I64; fp32 variant
              U[0,1) with SUM_F32.  Fixed-children reading N = 2^29 (the
              paper's 512M integers).
  D3 graph  : R-MAT scale 24 (Graph500 a,b,c,d = .57,.19,.19,.05, edge factor
              16, random vertex relabel), edges grouped by source vertex (CSR),
              u32 weights i.i.d. uniform; LT(2^31) filter, COUNT_MIN_U32.
  D4 text   : i.i.d. bytes: '\n' with p = 1/1397 (geometric lines of mean
              1397 chars), '{' with p = 45/1397 (~45 per line,
              P:681-682), digits with p = 1/2, other printable bytes
              otherwise; lines are CSR regions ending with their '\n'
              (reading A20); CLASS('{') filter, COUNT_XOR64.
  D5 zipf   : lengths Zipf(s=1.2) on [1, 4096], int32, sweep filters, SUM_I64.
"""
from __future__ import annotations

import numpy as np

# Odd multipliers for the HASH_LT filters (reading A13 of SURVEY §8(c)).
HASH_A = (0x9E3779B1, 0x85EBCA6B, 0xC2B2AE35, 0x27D4EB2F)
HASH_T = 192                      # keep ~3/4 per stage


def sweep_stages(n: int = 3, T: int = HASH_T):
    return [("hash_lt", HASH_A[k], T) for k in range(n)]


def tiny_stages():
    return sweep_stages(2)


def class_table(chars: bytes) -> bytes:
    """32-byte bitmap of a byte class (CLASS filter)."""
    t = bytearray(32)
    for c in chars:
        t[c >> 3] |= 1 << (c & 7)
    return bytes(t)


TEXT_CLASS = class_table(b"{")
_OTHER = np.frombuffer(b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ,.:;-_ }[]\"/=+", np.uint8)


def text_stages():
    return [("class", TEXT_CLASS)]


# ----------------------------------------------------------------- numpy side
def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def lengths(R: int, dist: str, L: int = 0, seed: int = 0, lo: int = 0, hi: int = 0,
            zipf_s: float = 1.2, zipf_max: int = 4096) -> np.ndarray:
    """Region lengths (int64[R]).
    dist: "fixed" (all L) | "var" (U{0..2L}, mean L; the paper's
    uniform-in-[0,max] with max = 2L) | "uniform" (U{lo..hi}) |
    "zipf" (P(k) ~ k^-s on [1, zipf_max])."""
    g = _rng(seed)
    if dist == "fixed":
        return np.full(R, L, np.int64)
    if dist == "var":
        return g.integers(0, 2 * L, size=R, endpoint=True, dtype=np.int64)
    if dist == "uniform":
        return g.integers(lo, hi, size=R, endpoint=True, dtype=np.int64)
    if dist == "zipf":
        k = np.arange(1, zipf_max + 1, dtype=np.float64)
        cdf = np.cumsum(k ** -zipf_s)
        cdf /= cdf[-1]
        u = g.random(R)
        return (np.searchsorted(cdf, u, side="right") + 1).clip(1, zipf_max).astype(np.int64)
    raise ValueError(dist)


def offsets(lens: np.ndarray, base: int = 0) -> np.ndarray:
    """CSR offsets int64[R+1] with offsets[0] = base."""
    off = np.empty(lens.size + 1, np.int64)
    off[0] = base
    np.cumsum(lens, out=off[1:])
    off[1:] += base
    return off


def values(N: int, dtype: str, seed: int = 0) -> np.ndarray:
    """Element values: i32/u32 full range, f32 U[0,1), u8 full range."""
    g = _rng(seed)
    if dtype == "i32":
        return g.integers(-2**31, 2**31, size=N, dtype=np.int64).astype(np.int32)
    if dtype == "u32":
        return g.integers(0, 2**32, size=N, dtype=np.uint64).astype(np.uint32)
    if dtype == "f32":
        return g.random(N, dtype=np.float32)
    if dtype == "u8":
        return g.integers(0, 256, size=N, dtype=np.uint8)
    raise ValueError(dtype)


def text(N: int, seed: int = 0, line_mean: float = 1397.0, brace_per_line: float = 45.0, base: int = 0):
    """D4 byte stream (numpy).  Returns (bytes u8[N], offsets int64[R+1]) with
    every line ending at its newline; a final unterminated line is a region."""
    g = _rng(seed)
    u = g.random(N)
    p_nl = 1.0 / line_mean
    p_br = brace_per_line / line_mean
    b = np.empty(N, np.uint8)
    other = _OTHER[g.integers(0, _OTHER.size, size=N)]
    digits = (ord("0") + g.integers(0, 10, size=N)).astype(np.uint8)
    b[:] = np.where(u < 0.5, digits, other)
    b[u < p_br + p_nl] = ord("{")
    b[u < p_nl] = ord("\n")
    nl = np.nonzero(b == ord("\n"))[0] + 1
    ends = nl if (nl.size and nl[-1] == N) else np.concatenate([nl, [N]])
    off = np.concatenate([[0], ends]).astype(np.int64) + base
    return b, off


def taxi(n_lines: int, seed: int = 0, pairs_mean: int = 45, line_mean: int = 1397):
    """Taxi-like corpus (lines of text holding "{x,y}" coordinate
    pairs, ~45 pairs and ~1397 chars per line).  The filler between pairs is
    letters and spaces only, so every '{' is a generated pair start.  About
    10% of the pairs are malformed ("{x;y}", "{x,}", "{,y}", "{x,y" at the line
    end, 10-digit fields); "{{x,y}" holds one well-formed pair.  Returns
    (bytes u8[N], offsets int64[R+1], expected) where expected lists
    (line, y, x) of every well-formed pair in stream order -- the second
    stage's result by construction."""
    g = _rng(seed)
    letters = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz      ", np.uint8)
    out, offs, exp = [], [0], []
    pos = 0
    for ln in range(n_lines):
        k = int(g.poisson(pairs_mean))
        fill = max(1, (line_mean - 14 * k) // (k + 1))
        parts = []
        for i in range(k + 1):
            parts.append(letters[g.integers(0, letters.size, int(g.integers(1, 2 * fill + 1)))].tobytes())
            if i == k:
                break
            x, y = int(g.integers(0, 10 ** int(g.integers(1, 7)))), int(g.integers(0, 10 ** int(g.integers(1, 7))))
            kind = int(g.integers(0, 100))
            if kind < 90:
                parts.append(b"{%d,%d}" % (x, y))
                exp.append((ln, y, x))
            elif kind < 92:
                parts.append(b"{%d;%d}" % (x, y))
            elif kind < 94:
                parts.append(b"{%d,}" % x)
            elif kind < 96:
                parts.append(b"{,%d}" % y)
            elif kind < 98:
                parts.append(b"{%d,%d}" % (x + 10 ** 9, y))          # 10-digit field
            else:
                parts.append(b"{{%d,%d}" % (x, y))
                exp.append((ln, y, x))
        if ln % 17 == 5 and k > 0:                                    # a pair cut by the line end
            parts.append(b"{%d,%d" % (7, 8))
        line = b"".join(parts) + b"\n"
        out.append(line)
        pos += len(line)
        offs.append(pos)
    b = np.frombuffer(b"".join(out), np.uint8).copy()
    return b, np.array(offs, np.int64), np.array(exp, np.uint32).reshape(-1, 3)


def taxi_stages():
    return [("class", class_table(b"{"))]


def tiny(seed: int = 0x5EED + 1):
    """D1: 1000 parents, 1-64 children each, int32, 2 int filters, SUM_I64."""
    lens = lengths(1000, "uniform", lo=1, hi=64, seed=seed)
    off = offsets(lens)
    return values(int(off[-1]), "i32", seed + 17), off, tiny_stages(), "sum_i64"


# ----------------------------------------------------------------- torch side
def torch_lengths(R: int, dist: str, L: int = 0, seed: int = 0, device="cuda",
                  zipf_s: float = 1.2, zipf_max: int = 4096, lo: int = 0, hi: int = 0):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if dist == "fixed":
        return torch.full((R,), L, dtype=torch.int64, device=device)
    if dist == "var":
        return torch.randint(0, 2 * L + 1, (R,), generator=g, device=device, dtype=torch.int64)
    if dist == "uniform":
        return torch.randint(lo, hi + 1, (R,), generator=g, device=device, dtype=torch.int64)
    if dist == "zipf":
        k = torch.arange(1, zipf_max + 1, dtype=torch.float64, device=device)
        cdf = torch.cumsum(k ** -zipf_s, 0)
        cdf /= cdf[-1].clone()
        u = torch.rand(R, generator=g, device=device, dtype=torch.float64)
        return (torch.searchsorted(cdf, u, right=True) + 1).clamp(1, zipf_max).to(torch.int64)
    raise ValueError(dist)


def torch_offsets(lens, base: int = 0):
    import torch
    off = torch.empty(lens.numel() + 1, dtype=torch.int64, device=lens.device)
    off[0] = base
    torch.cumsum(lens, 0, out=off[1:])
    if base:
        off[1:] += base
    return off


def torch_values(N: int, dtype: str, seed: int = 0, device="cuda"):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if dtype == "i32":
        return torch.randint(-2**31, 2**31, (N,), generator=g, device=device, dtype=torch.int64).to(torch.int32) \
            if N <= 2**24 else _torch_bits(N, g, device).view(torch.int32)
    if dtype == "u32":
        return _torch_bits(N, g, device).view(torch.int32)        # raw bits; reinterpret as u32
    if dtype == "f32":
        return torch.rand(N, generator=g, device=device, dtype=torch.float32)
    if dtype == "u8":
        return torch.randint(0, 256, (N,), generator=g, device=device, dtype=torch.uint8)
    raise ValueError(dtype)


def torch_text(N: int, seed: int = 0, device="cuda", line_mean: float = 1397.0, brace_per_line: float = 45.0):
    """D4 byte stream generated on the device (same recipe as text())."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = torch.rand(N, generator=g, device=device, dtype=torch.float32)
    other = torch.from_numpy(_OTHER.copy()).to(device)
    pick = torch.randint(0, other.numel(), (N,), generator=g, device=device, dtype=torch.int32)
    digit = torch.randint(ord("0"), ord("9") + 1, (N,), generator=g, device=device, dtype=torch.int32).to(torch.uint8)
    b = torch.where(u < 0.5, digit, other[pick])
    p_nl = 1.0 / line_mean
    b[u < p_nl + brace_per_line / line_mean] = ord("{")
    b[u < p_nl] = ord("\n")
    del u, pick, digit
    nl = torch.nonzero(b == ord("\n")).flatten().to(torch.int64) + 1
    if nl.numel() == 0 or int(nl[-1].item()) != N:
        nl = torch.cat([nl, torch.tensor([N], dtype=torch.int64, device=device)])
    off = torch.cat([torch.zeros(1, dtype=torch.int64, device=device), nl])
    return b, off


def torch_rmat_csr(scale: int = 24, edge_factor: int = 16, seed: int = 0, device="cuda",
                   a: float = 0.57, b: float = 0.19, c: float = 0.19):
    """D3: R-MAT source-vertex degrees -> CSR offsets (int64[V+1]) plus u32
    edge weights (returned as an int32 view) per CSR slot.  Only the source of
    each edge matters for grouping; its bit at every level is 1 with
    probability c + d (the lower two quadrants), independently per level."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    V = 1 << scale
    E = edge_factor * V
    p1 = 1.0 - a - b                       # P(source bit = 1) = c + d
    src = torch.zeros(E, dtype=torch.int64, device=device)
    for lvl in range(scale):
        bit = (torch.rand(E, generator=g, device=device) < p1).to(torch.int64)
        src |= bit << lvl
    perm = torch.randperm(V, generator=g, device=device)
    deg = torch.bincount(perm[src], minlength=V)
    del src
    off = torch_offsets(deg)
    w = _torch_bits(E, g, device).view(torch.int32)
    return w, off


def _torch_bits(N: int, g, device):
    import torch
    # 32 random bits per element from two 16-bit draws (int32 randint range limits)
    hi = torch.randint(0, 1 << 16, (N,), generator=g, device=device, dtype=torch.int32)
    lo = torch.randint(0, 1 << 16, (N,), generator=g, device=device, dtype=torch.int32)
    return (hi << 16) | lo
