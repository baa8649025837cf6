"""Python big-integer micro-oracle of the LSHBloom hot path (test infrastructure only).

A second, from-scratch implementation of the conventions DESIGN.md section 3 writes down
(R1 fingerprint, R3 truncate-then-min, R4 exact arithmetic, R5 counter-mode family, R6 band
hash, R9 sizing, R10 probe positions, R11 bit layout, R12/R13 stream order) and of the blocked
variant's offsets.  It was written from those prose definitions, not from
oracle/lshbloom_oracle.c, and uses only Python integers (arbitrary precision: no 2^64 or 2^128
wrap anywhere except where a convention says "wraps mod 2^64"), so a misreading in the C oracle
-- `h + w` for `h ^ w`, the salt taken from the shingle count instead of its length, `a_i` drawn
from counter 2i+1 instead of 2i, an off-by-one in a 10-bit field -- shows up as a mismatch in
tests/test_oracle_micro.py.  It is slow (pure-Python loops) and meant for tiny inputs.

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
from __future__ import annotations

import math

M64 = (1 << 64) - 1
P = (1 << 61) - 1                        # the Mersenne prime 2^61 - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15        # SplitMix64 increment
FP_SALT = 0x6C7368626C6F6F6D             # ASCII "lshbloom" read as a big-endian u64 (DESIGN R1)


def splitmix64_finaliser(z: int) -> int:
    """DESIGN R5: z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27; z *= 0x94D049BB133111EB;
    z ^= z>>31 -- every step mod 2^64."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def counter_draw(seed: int, domain: int, i: int) -> int:
    """R(seed, dom, i) = mix64(seed + gamma * (dom * 2^32 + i + 1)), the sum wrapping mod 2^64."""
    return splitmix64_finaliser(seed + GOLDEN_GAMMA * (domain * 2**32 + i + 1))


def permutation_coefficients(seed: int, num_perm: int):
    """a_i = 1 + R(seed,1,2i) mod (P-1), b_i = R(seed,1,2i+1) mod P."""
    a = [1 + counter_draw(seed, 1, 2 * i) % (P - 1) for i in range(num_perm)]
    b = [counter_draw(seed, 1, 2 * i + 1) % P for i in range(num_perm)]
    return a, b


def band_coefficients(seed: int, r: int):
    """c_u = 1 + R(seed,2,2u) mod (P-1), d_u = R(seed,2,2u+1) mod P (DESIGN R5/R6)."""
    c = [1 + counter_draw(seed, 2, 2 * u) % (P - 1) for u in range(r)]
    d = [counter_draw(seed, 2, 2 * u + 1) % P for u in range(r)]
    return c, d


def filter_seeds(seed: int, bands):
    """s1_j = R(seed,3,j), s2_j = R(seed,4,j) for the GLOBAL band indices j."""
    return [counter_draw(seed, 3, j) for j in bands], [counter_draw(seed, 4, j) for j in bands]


def shingle_fingerprint(ids) -> int:
    """DESIGN R1: h = mix64(salt + t) with t the shingle's length in ids, then for each id w in
    order h = mix64(h XOR w)."""
    h = splitmix64_finaliser(FP_SALT + len(ids))
    for w in ids:
        h = splitmix64_finaliser(h ^ (int(w) & 0xFFFFFFFF))
    return h


def shingles(ids, n: int = 5):
    """Every contiguous n-gram; a document shorter than n is one shingle."""
    ids = [int(w) for w in ids]
    if not ids:
        raise ValueError("empty document")
    if len(ids) < n:
        return [tuple(ids)]
    return [tuple(ids[q:q + n]) for q in range(len(ids) - n + 1)]


def signature(ids, num_perm: int, seed: int, n: int = 5):
    """sig[i] = min over the shingle SET of ((a_i x + b_i) mod P) mod 2^32, x = fp mod P
    (DESIGN R3 truncate-then-min, R4 exact)."""
    a, b = permutation_coefficients(seed, num_perm)
    xs = {shingle_fingerprint(s) % P for s in shingles(ids, n)}
    return [min(((a[i] * x + b[i]) % P) % 2**32 for x in xs) for i in range(num_perm)]


def band_hash(sig, j: int, r: int, seed: int) -> int:
    """BH_j = (sum_{u<r} (c_u sig[j r + u] + d_u) mod P) mod P."""
    c, d = band_coefficients(seed, r)
    return sum((c[u] * sig[j * r + u] + d[u]) % P for u in range(r)) % P


def bloom_geometry(n_expected: int, p: float):
    """m = ceil(-n ln p / (ln 2)^2), k = max(1, round-half-away((m / n) ln 2)) (R9)."""
    m = math.ceil(-float(n_expected) * math.log(p) / (math.log(2.0) * math.log(2.0)))
    kf = (m / float(n_expected)) * math.log(2.0)
    k = int(math.floor(kf + 0.5))                    # llround for positive values
    return int(m), max(1, k)


def probe_hashes(bh: int, s1: int, s2: int):
    """h1 = mix64(BH xor s1_j), h2 = mix64(BH xor s2_j) | 1 (R10)."""
    return splitmix64_finaliser(bh ^ s1), splitmix64_finaliser(bh ^ s2) | 1


def probe_positions(bh: int, s1: int, s2: int, m: int, k: int):
    """g_t = (h1 + t h2) mod m over the integers, t < k (R10; 0-based positions)."""
    h1, h2 = probe_hashes(bh, s1, s2)
    return [(h1 + t * h2) % m for t in range(k)]


def blocked_positions(bh: int, s1: int, s2: int, n_blocks: int, k: int):
    """Blocked variant: block = h1 mod nb; offset_t = bits
    [10 (t mod 6), 10 (t mod 6) + 10) of mix64(h2 + floor(t / 6)) (the sum wrapping mod 2^64);
    g_t = 1024 block + offset_t."""
    h1, h2 = probe_hashes(bh, s1, s2)
    block = h1 % n_blocks
    out = []
    for t in range(k):
        word = splitmix64_finaliser(h2 + t // 6)
        field = (word >> (10 * (t % 6))) % 1024
        out.append(1024 * block + field)
    return out


class BloomIndex:
    """b Bloom filters, one per band, each a Python set of set-bit positions;
    documents are processed one at a time in stream order: query all k bits, then set them
    (insert unconditional: R12)."""

    def __init__(self, b: int, n_expected: int, p: float, seed: int, blocked: bool = False):
        self.b, self.seed, self.blocked = b, seed, blocked
        self.m, self.k = bloom_geometry(n_expected, p)
        if blocked:
            self.n_blocks = -(-self.m // 1024)
            self.m = 1024 * self.n_blocks
        self.s1, self.s2 = filter_seeds(seed, range(b))
        self.bits = [set() for _ in range(b)]

    def positions(self, j: int, bh: int):
        if self.blocked:
            return blocked_positions(bh, self.s1[j], self.s2[j], self.n_blocks, self.k)
        return probe_positions(bh, self.s1[j], self.s2[j], self.m, self.k)

    def query_insert_doc(self, bhs):
        """bhs = the document's b band hashes; returns (dup, per-band hits)."""
        hits = []
        for j, bh in enumerate(bhs):
            pos = self.positions(j, bh)
            hits.append(all(g in self.bits[j] for g in pos))
            self.bits[j].update(pos)
        return any(hits), hits

    def filter_bytes(self, j: int) -> bytes:
        """The filter as S:322's little-endian payload: bit g in byte g >> 3 at mask 1 << (g & 7)."""
        buf = bytearray((self.m + 7) // 8)
        for g in self.bits[j]:
            buf[g >> 3] |= 1 << (g & 7)
        return bytes(buf)


def run(docs, *, num_perm: int, b: int, r: int, n_expected: int, p: float, seed: int, n: int = 5,
        blocked: bool = False):
    """Signatures, band hashes and duplicate flags of a list of documents (lists of ids)."""
    idx = BloomIndex(b, n_expected, p, seed, blocked)
    sigs, bhs, dups = [], [], []
    for ids in docs:
        sig = signature(ids, num_perm, seed, n)
        bh = [band_hash(sig, j, r, seed) for j in range(b)]
        dup, _ = idx.query_insert_doc(bh)
        sigs.append(sig)
        bhs.append(bh)
        dups.append(int(dup))
    return sigs, bhs, dups, idx
