"""Seeded synthetic batches shaped like the paper's ADEPT workloads.

This module holds NO alignment arithmetic: it only draws sequences.  It is the
one module both sides use -- the CPU oracle (``oracle/``) and the CUDA path
receive the very same bytes from it (DESIGN.md sec. "Input recipe").

The paper's data (30,000 + 4.6 M ADEPT DNA pairs) is not
available, so each BASELINE.json config is realised as a seeded synthetic
batch:

* DNA: i.i.d. uniform ACGT.  90 % of pairs are *related*: the reference embeds
  the read mutated with 2 % substitutions, 0.5 % insertions and 0.5 %
  deletions, at a random offset between random flanks, truncated to m.  The
  other 10 % are unrelated random references.
* Protein: i.i.d. uniform over the 20 standard residues; 70 % related (30 %
  substitutions, 2 % insertions, 2 % deletions), 30 % unrelated.

Pairs are generated in blocks of ``BLOCK`` pairs.  Block b of config k draws
its lengths from ``SeedSequence([220812350 + k, b, 0])`` and its residues from
``SeedSequence([220812350 + k, b, 1])``, so any sub-range of a batch (one
rank's shard) and the lengths of the whole batch (for the cell-count shard
plan) can be produced without generating everything.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BLOCK = 1024
SEED_BASE = 220812350

DNA_ALPHA = np.frombuffer(b"ACGT", dtype=np.uint8)
PROT_ALPHA = np.frombuffer(b"ARNDCQEGHILKMFPSTWYV", dtype=np.uint8)

DNA_SCORING = {"alphabet": "dna", "match": 3, "mismatch": -3, "gap_open": -6, "gap_extend": -1}
PROTEIN_SCORING = {"alphabet": "protein", "match": 0, "mismatch": 0, "gap_open": -11, "gap_extend": -1}


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config realised as a synthetic batch recipe."""
    index: int               # k in SEED_BASE + k (1-based, BASELINE.json configs[k-1])
    name: str
    alphabet: str            # 'dna' | 'protein'
    n_pairs: int
    scoring: dict
    # length model: 'fixed_q' (n fixed, m uniform), 'indep' (n, m uniform),
    # 'mixed' (C5: short fraction + log-uniform long pairs)
    lengths: str
    n_fixed: int = 150
    n_range: tuple = (150, 150)
    m_range: tuple = (150, 1024)
    long_frac: float = 0.0
    long_n: tuple = (150, 4096)
    long_m: tuple = (1024, 16384)
    related: float = 0.9
    sub: float = 0.02
    ins: float = 0.005
    dele: float = 0.005
    baseline_text: str = ""
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "c1": Config(1, "c1_dna_1k_150x300", "dna", 1000, DNA_SCORING, "fixed_q", m_range=(150, 300),
                 baseline_text="1,000 synthetic DNA pairs, query 150 bp vs reference <=300 bp, "
                               "match 3 / mismatch -3 / gap open -6 / extend -1, score+end+start, 1 GPU"),
    "c2": Config(2, "c2_dna_100k_150x1024", "dna", 100_000, DNA_SCORING, "fixed_q", m_range=(150, 1024),
                 baseline_text="ADEPT-shaped DNA batch: 100k pairs, 150 bp reads vs contigs up to 1,024 bp, 1 B200"),
    "c3": Config(3, "c3_protein_50k_1024", "protein", 50_000, PROTEIN_SCORING, "indep",
                 n_range=(32, 1024), m_range=(32, 1024), related=0.7, sub=0.30, ins=0.02, dele=0.02,
                 baseline_text="protein batch BLOSUM62 with affine gaps, 50k pairs with lengths up to 1,024 residues, 1 B200"),
    "c4": Config(4, "c4_dna_4m_150x1024", "dna", 4_000_000, DNA_SCORING, "fixed_q", m_range=(150, 1024),
                 baseline_text="DNA batch of 4M pairs sharded by cell count across 1/2/4/8 B200"),
    "c5": Config(5, "c5_dna_400k_mixed_16kb", "dna", 400_000, DNA_SCORING, "mixed", m_range=(150, 1024),
                 long_frac=0.3, long_n=(150, 4096), long_m=(1024, 16384),
                 baseline_text="length-skewed mixed batch with references up to 16 kb "
                               "(multi-tile striped wavefront, load balance), 8 B200"),
}


@dataclass
class Batch:
    """CSR batch: pair p is queries[q_offsets[p]:q_offsets[p+1]] vs refs[r_offsets[p]:r_offsets[p+1]]."""
    queries: np.ndarray    # uint8 ASCII
    q_offsets: np.ndarray  # int64, n_pairs + 1
    refs: np.ndarray       # uint8 ASCII
    r_offsets: np.ndarray  # int64, n_pairs + 1
    scoring: dict
    name: str = ""

    @property
    def n_pairs(self) -> int:
        return int(self.q_offsets.size - 1)

    def lengths(self):
        return np.diff(self.q_offsets), np.diff(self.r_offsets)

    def cells(self) -> int:
        n, m = self.lengths()
        return int(np.sum(n.astype(np.int64) * m.astype(np.int64)))

    def pair(self, p: int):
        return (bytes(self.queries[self.q_offsets[p]:self.q_offsets[p + 1]]),
                bytes(self.refs[self.r_offsets[p]:self.r_offsets[p + 1]]))

    def subset(self, idx) -> "Batch":
        return from_pairs([self.pair(int(p)) for p in idx], self.scoring, self.name + "_subset")


def from_pairs(pairs, scoring, name="pairs") -> Batch:
    """Build a Batch from a list of (query, reference) str/bytes."""
    qs = [p[0].encode() if isinstance(p[0], str) else bytes(p[0]) for p in pairs]
    rs = [p[1].encode() if isinstance(p[1], str) else bytes(p[1]) for p in pairs]
    qo = np.zeros(len(pairs) + 1, dtype=np.int64)
    ro = np.zeros(len(pairs) + 1, dtype=np.int64)
    qo[1:] = np.cumsum([len(x) for x in qs]) if qs else []
    ro[1:] = np.cumsum([len(x) for x in rs]) if rs else []
    qa = np.frombuffer(b"".join(qs), dtype=np.uint8).copy() if qs else np.zeros(0, np.uint8)
    ra = np.frombuffer(b"".join(rs), dtype=np.uint8).copy() if rs else np.zeros(0, np.uint8)
    return Batch(qa, qo, ra, ro, dict(scoring), name)


def _block_lengths(cfg: Config, b: int, count: int):
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE + cfg.index, b, 0])))
    if cfg.lengths == "fixed_q":
        n = np.full(count, cfg.n_fixed, dtype=np.int64)
        m = rng.integers(cfg.m_range[0], cfg.m_range[1] + 1, size=count, dtype=np.int64)
    elif cfg.lengths == "indep":
        n = rng.integers(cfg.n_range[0], cfg.n_range[1] + 1, size=count, dtype=np.int64)
        m = rng.integers(cfg.m_range[0], cfg.m_range[1] + 1, size=count, dtype=np.int64)
    elif cfg.lengths == "mixed":
        is_long = rng.random(count) < cfg.long_frac
        n_s = np.full(count, cfg.n_fixed, dtype=np.int64)
        m_s = rng.integers(cfg.m_range[0], cfg.m_range[1] + 1, size=count, dtype=np.int64)
        ln = np.log(cfg.long_n)
        lm = np.log(cfg.long_m)
        n_l = np.floor(np.exp(rng.uniform(ln[0], ln[1], size=count))).astype(np.int64)
        m_l = np.floor(np.exp(rng.uniform(lm[0], lm[1], size=count))).astype(np.int64)
        n = np.where(is_long, np.clip(n_l, cfg.long_n[0], cfg.long_n[1]), n_s)
        m = np.where(is_long, np.clip(m_l, cfg.long_m[0], cfg.long_m[1]), m_s)
    else:
        raise ValueError(cfg.lengths)
    return n, m


def batch_lengths(cfg: Config, start: int = 0, stop: int | None = None):
    """Lengths (n, m) of pairs [start, stop) without drawing residues."""
    stop = cfg.n_pairs if stop is None else stop
    ns, ms = [], []
    for b in range(start // BLOCK, (stop + BLOCK - 1) // BLOCK):
        lo, hi = b * BLOCK, min((b + 1) * BLOCK, cfg.n_pairs)
        n, m = _block_lengths(cfg, b, hi - lo)
        s0, s1 = max(start, lo) - lo, min(stop, hi) - lo
        ns.append(n[s0:s1]); ms.append(m[s0:s1])
    if not ns:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(ns), np.concatenate(ms)


def _mutate(rng, seq: np.ndarray, alpha: np.ndarray, sub: float, ins: float, dele: float) -> np.ndarray:
    L = seq.size
    out = seq.copy()
    # substitutions to a different symbol
    smask = rng.random(L) < sub
    if smask.any():
        k = int(smask.sum())
        shift = rng.integers(1, alpha.size, size=k)
        lut = np.zeros(256, np.int64)
        lut[alpha] = np.arange(alpha.size)
        out[smask] = alpha[(lut[out[smask]] + shift) % alpha.size]
    keep = rng.random(L) >= dele
    insm = rng.random(L) < ins
    pieces_len = keep.astype(np.int64) + insm.astype(np.int64)
    total = int(pieces_len.sum())
    res = np.empty(total, dtype=np.uint8)
    pos = np.cumsum(pieces_len) - pieces_len
    res[pos[keep]] = out[keep]
    ins_pos = pos[insm] + keep[insm].astype(np.int64)
    res[ins_pos] = alpha[rng.integers(0, alpha.size, size=ins_pos.size)]
    return res


def _gen_block(cfg: Config, b: int, count: int):
    n, m = _block_lengths(cfg, b, count)
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE + cfg.index, b, 1])))
    alpha = DNA_ALPHA if cfg.alphabet == "dna" else PROT_ALPHA
    alpha_sorted = np.sort(alpha)
    qs, rs = [], []
    rel = rng.random(count) < cfg.related
    for p in range(count):
        q = alpha[rng.integers(0, alpha.size, size=int(n[p]))]
        mm = int(m[p])
        if rel[p]:
            mut = _mutate(rng, q, alpha_sorted, cfg.sub, cfg.ins, cfg.dele)
            if mut.size >= mm:
                s = int(rng.integers(0, mut.size - mm + 1))
                r = mut[s:s + mm]
            else:
                r = alpha[rng.integers(0, alpha.size, size=mm)]
                off = int(rng.integers(0, mm - mut.size + 1))
                r[off:off + mut.size] = mut
        else:
            r = alpha[rng.integers(0, alpha.size, size=mm)]
        qs.append(q); rs.append(r)
    return n, m, qs, rs


def generate(cfg: Config | str, start: int = 0, stop: int | None = None) -> Batch:
    """Pairs [start, stop) of config ``cfg`` (a Config or a key of CONFIGS)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    stop = cfg.n_pairs if stop is None else min(stop, cfg.n_pairs)
    qs, rs = [], []
    for b in range(start // BLOCK, (stop + BLOCK - 1) // BLOCK):
        lo, hi = b * BLOCK, min((b + 1) * BLOCK, cfg.n_pairs)
        _, _, bq, br = _gen_block(cfg, b, hi - lo)
        s0, s1 = max(start, lo) - lo, min(stop, hi) - lo
        qs.extend(bq[s0:s1]); rs.extend(br[s0:s1])
    qo = np.zeros(len(qs) + 1, dtype=np.int64)
    ro = np.zeros(len(rs) + 1, dtype=np.int64)
    if qs:
        qo[1:] = np.cumsum([x.size for x in qs])
        ro[1:] = np.cumsum([x.size for x in rs])
    qa = np.concatenate(qs) if qs else np.zeros(0, np.uint8)
    ra = np.concatenate(rs) if rs else np.zeros(0, np.uint8)
    return Batch(qa.astype(np.uint8), qo, ra.astype(np.uint8), ro, dict(cfg.scoring), f"{cfg.name}[{start}:{stop}]")


def _gen_range(args):
    key, start, stop = args
    b = generate(key, start, stop)
    return b.queries, np.diff(b.q_offsets), b.refs, np.diff(b.r_offsets)


def generate_parallel(cfg: Config | str, start: int = 0, stop: int | None = None, workers: int | None = None) -> Batch:
    """generate() split over worker processes by whole blocks: byte-identical to generate(cfg, start,
    stop) (every block draws from its own seed), for the large configs (c4: 4 M pairs)."""
    import multiprocessing as mp
    import os
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    stop = cfg.n_pairs if stop is None else min(stop, cfg.n_pairs)
    workers = workers or min(32, os.cpu_count() or 1)
    if workers <= 1 or stop - start <= 4 * BLOCK:
        return generate(cfg, start, stop)
    key = next(k for k, v in CONFIGS.items() if v is cfg)
    step = max(BLOCK, ((stop - start) // (4 * workers) + BLOCK - 1) // BLOCK * BLOCK)
    cuts = list(range(start, stop, step)) + [stop]
    jobs = [(key, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    with mp.get_context("fork").Pool(workers) as pool:
        parts = pool.map(_gen_range, jobs)
    n = np.concatenate([p[1] for p in parts])
    m = np.concatenate([p[3] for p in parts])
    qo = np.zeros(n.size + 1, np.int64)
    ro = np.zeros(m.size + 1, np.int64)
    qo[1:] = np.cumsum(n)
    ro[1:] = np.cumsum(m)
    return Batch(np.concatenate([p[0] for p in parts]), qo, np.concatenate([p[2] for p in parts]), ro,
                 dict(cfg.scoring), f"{cfg.name}[{start}:{stop}]")


def batch_sha256(b: Batch) -> str:
    """SHA-256 over the batch's CSR arrays and scoring (the reproducibility record of SURVEY 8(d))."""
    import hashlib
    import json
    h = hashlib.sha256()
    for arr in (b.q_offsets, b.queries, b.r_offsets, b.refs):
        h.update(np.ascontiguousarray(arr).tobytes())
    h.update(json.dumps(b.scoring, sort_keys=True).encode())
    return h.hexdigest()


def random_pairs(seed: int, count: int, n_range, m_range, alphabet: bytes = b"ACGT", scoring=None,
                 name="random") -> Batch:
    """Unrelated i.i.d. pairs over ``alphabet`` (tests: tiny/adversarial sets)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE, 7, seed])))
    alpha = np.frombuffer(alphabet, dtype=np.uint8)
    pairs = []
    for _ in range(count):
        n = int(rng.integers(n_range[0], n_range[1] + 1))
        m = int(rng.integers(m_range[0], m_range[1] + 1))
        pairs.append((alpha[rng.integers(0, alpha.size, size=n)].tobytes(),
                      alpha[rng.integers(0, alpha.size, size=m)].tobytes()))
    return from_pairs(pairs, scoring or DNA_SCORING, name)


# ------------------------------------------------------------ SIMCoV diffusion fields (f4)

SIMCOV_HELDOUT = (2500, 2500)  # the held-out grid of PAPER.md:567 ("a larger grid size: 2500x2500")


def simcov_fields(seed: int, H: int, W: int, n_fields: int = 2, sites: int | None = None,
                  peak: int = 1 << 24, background: float = 0.0):
    """Seeded SIMCoV-shaped concentration fields (uint32 H x W arrays, one per field).

    SIMCoV seeds a lung-tissue grid with "a set of infection sites" from which virions and
    inflammatory signal spread: each field is zero except at ``sites``
    random points (default: one per 10,000 cells, at least 1) holding a concentration drawn
    uniformly from [peak/2, peak), plus, if ``background`` > 0, that fraction of cells
    holding a uniform value below peak/64 (an established, already-spread infection).
    No diffusion arithmetic here: the same arrays go to the oracle and the CUDA path.
    """
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE, 22, seed])))
    cells = H * W
    k = max(1, cells // 10000) if sites is None else sites
    out = []
    for _ in range(n_fields):
        f = np.zeros(cells, np.uint32)
        if cells:
            if background > 0:
                nb = int(cells * background)
                f[rng.integers(0, cells, size=nb)] = rng.integers(0, max(1, peak // 64), size=nb, dtype=np.uint32)
            f[rng.integers(0, cells, size=min(k, cells))] = rng.integers(peak // 2, peak, size=min(k, cells),
                                                                         dtype=np.uint32)
        out.append(f.reshape(H, W))
    return out


def simcov_dense(seed: int, H: int, W: int, n_fields: int = 2, high: int = 1 << 31):
    """Seeded uniform fields in [0, high) (tests: full-range arithmetic, every cell active)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE, 23, seed])))
    return [rng.integers(0, high, size=(H, W), dtype=np.uint64).astype(np.uint32) for _ in range(n_fields)]
