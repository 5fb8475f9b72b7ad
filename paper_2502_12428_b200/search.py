"""Drop-in for the reference's batch and search drivers (qfsplit/search.py) on the B200 engine.

Same names, configuration, results and determinism contract as the reference:

    SearchConfig, HeightHistogram, FoundSurface       search.py:23-89
    sample_surface(rng, p, n=4)                       search.py:92-98   (one rng.integers(0,p,35) per attempt)
    run_search(cfg)                                   search.py:121-154 (blocks per worker, (seed, worker) streams)
    parse_fixtures / verify_fixtures                  search.py:181-229
    histogram_text / found_surfaces_text              search.py:232-251

A reference "worker" (a process of its ProcessPoolExecutor) becomes a GPU worker here: worker w
draws its whole block from `default_rng([seed, w])` exactly as search._worker_block does, and the
block's heights are computed in ONE batched call on device `devices[w % len(devices)]`.  The
histogram and the found-log for a given (seed, parallelism) are therefore identical to the
reference's; `target_height` keeps the reference's per-worker semantics (a worker's record stops
at its first sample of that height).

New on top: `spectrum_search` keeps sampling seeded blocks until every
height 1..bound and infinity has been seen, and returns one witness per height in fixture-table
format.
"""
from __future__ import annotations

import math
import threading
from dataclasses import dataclass, field

import numpy as np

from .errors import DomainError, ParseError
from .height import (INFINITE, HeightResult, SurfaceProblem, decode_height, default_bound, height_batch,
                     height_matrix, split_blocks, is_prime)
from .quartic import NCOEFF, NVARS, Quartic, parse_poly, poly_to_text


@dataclass(frozen=True)
class SearchConfig:
    p: int
    n: int = 4
    sample_count: int = 1000
    rng_seed: int = 0
    bound: int | None = None
    target_height: int | None = None
    parallelism: int = 1

    def __post_init__(self):
        if self.sample_count < 1:
            raise DomainError(f"sample_count must be >= 1, got {self.sample_count}")
        if self.parallelism < 1:
            raise DomainError(f"parallelism must be >= 1, got {self.parallelism}")
        if self.target_height is not None and self.target_height < 1:
            raise DomainError("target_height must be a positive height")


@dataclass
class HeightHistogram:
    """Counts per finite height 1..bound plus infinity (search.py:42-80)."""

    bound: int
    counts: dict = field(default_factory=dict)
    infinite: int = 0
    total: int = 0

    def record(self, height):
        if isinstance(height, float) and math.isinf(height):
            self.infinite += 1
        else:
            self.counts[height] = self.counts.get(height, 0) + 1
        self.total += 1

    def record_codes(self, codes):
        """Bulk `record` of C-ABI height codes (int8 array, 0 = infinity)."""
        codes = np.asarray(codes)
        if codes.size == 0:
            return
        bc = np.bincount(codes.astype(np.int64), minlength=1)
        self.infinite += int(bc[0])
        for h in range(1, len(bc)):
            if bc[h]:
                self.counts[h] = self.counts.get(h, 0) + int(bc[h])
        self.total += int(codes.size)

    def merge(self, other: "HeightHistogram"):
        if other.bound != self.bound:
            raise DomainError("histograms cover different bounds")
        for h, c in other.counts.items():
            self.counts[h] = self.counts.get(h, 0) + c
        self.infinite += other.infinite
        self.total += other.total

    def fraction_at_least(self, h: int) -> float:
        hits = self.infinite + sum(c for k, c in self.counts.items() if k >= h)
        return hits / self.total if self.total else 0.0

    def as_dict(self) -> dict:
        return {"bound": self.bound, "counts": {str(h): self.counts[h] for h in sorted(self.counts)},
                "inf": self.infinite, "total": self.total}

    def check(self):
        if sum(self.counts.values()) + self.infinite != self.total:
            raise DomainError("histogram counts do not sum to total")


@dataclass(frozen=True)
class FoundSurface:
    """A sample that set a new maximum finite height when it was seen (search.py:83-89)."""

    index: int
    height: int
    f: Quartic


# ---- sampling (bit-identical stream consumption to search.py:92-98) ---------------------------------

def sample_coeffs(rng, p: int) -> np.ndarray:
    """One uniform nonzero coefficient vector: `rng.integers(0, p, size=35)` per attempt, zero draws redrawn."""
    while True:
        v = rng.integers(0, p, size=NCOEFF)
        if v.any():
            return v.astype(np.uint8)


def sample_surface(rng, p: int, n: int = 4) -> Quartic:
    if n != NVARS:
        raise DomainError(f"the GPU engine samples quartics in 4 variables; got n={n}")
    return Quartic(sample_coeffs(rng, p), p)


def sample_rows(rng, p: int, count: int) -> np.ndarray:
    """The next `count` samples of search.sample_surface drawn from `rng`, vectorised.

    `rng.integers(0, p, size=(m, 35))` consumes the bit stream exactly like m successive
    `rng.integers(0, p, size=35)` calls (numpy draws bounded int64 values one by one with no state carried
    between calls; pinned against the reference's own seeded dumps in tests/test_host_api.py), and the
    reference keeps the first nonzero draw of every attempt loop -- i.e. the samples are the draws with the
    all-zero rows (probability p^-35) removed.
    """
    out = np.empty((count, NCOEFF), dtype=np.uint8)
    have = 0
    while have < count:
        draws = rng.integers(0, p, size=(count - have, NCOEFF))
        keep = draws[draws.any(axis=1)]
        out[have:have + len(keep)] = keep
        have += len(keep)
    return out


def sample_block(p: int, count: int, seed: int, worker: int) -> np.ndarray:
    """The `count` coefficient vectors worker `worker` draws in search._worker_block (search.py:103,108)."""
    return sample_rows(np.random.default_rng([seed, worker]), p, count)


# ---- run_search -------------------------------------------------------------------------------------------

def _finish_block(cfg, start, coeffs, codes):
    """Histogram / found-log / best of one worker block from its height codes (search.py:104-118).  `coeffs` is anything
    indexable by row that yields the 35 coefficients (a numpy array, a torch tensor on the device)."""
    bound = cfg.bound if cfg.bound is not None else default_bound(cfg.n)
    used = len(codes)
    if cfg.target_height is not None:
        hits = np.nonzero(codes == cfg.target_height)[0]
        if hits.size:
            used = int(hits[0]) + 1  # the worker breaks right after recording its first hit
    codes = codes[:used]
    hist = HeightHistogram(bound)
    hist.record_codes(codes)
    found, best = [], 0
    finite = codes.astype(np.int64)
    # positions where the running maximum of the finite heights strictly increases
    run = np.maximum.accumulate(finite) if used else finite
    prev = np.concatenate(([0], run[:-1])) if used else run
    for i in np.nonzero((finite > prev) & (finite > 0))[0]:
        best = int(finite[i])
        found.append(FoundSurface(start + int(i), best, Quartic(_row(coeffs, int(i)), cfg.p)))
    return hist, found, best


def _row(coeffs, i):
    r = coeffs[i]
    return r.cpu().numpy() if hasattr(r, "cpu") else np.asarray(r)


def device_block(p: int, count: int, seed: int, worker: int, device: int = 0, bound: int = 10, method: str = "matrix"):
    """One worker block entirely on the GPU: the coefficient vectors are drawn on the device (csrc/qfs_sample.cuh: numpy's PCG64
    stream of default_rng([seed, worker]) jumped ahead per row), the heights are computed there, and only the height codes come
    back.  Returns (coeffs, codes, iters): coeffs is a torch CUDA tensor [count,35] (rows are fetched on demand), or a numpy array
    when the device reported a stream-shifting event (a Lemire rejection or a zero draw: about one block in 200 at 100 000
    rows) and the block was redrawn on the host -- either way the reference's samples, bit for bit."""
    from .engine import get_engine
    from .height import _check_engine_shape
    if not is_prime(p):
        raise DomainError(f"p={p} is not prime")
    _check_engine_shape(p)
    if method not in ("matrix", "naive", "lazy"):
        raise DomainError(f"unknown method {method!r}, expected 'matrix', 'naive' or 'lazy'")
    eng = get_engine(p, device)
    try:
        import torch   # only to own the device buffer of the block
    except ImportError:
        host, clean = eng.sample(seed, worker, count)          # still drawn on the device, returned to the host
        if not clean:
            host = sample_block(p, count, seed, worker)
        codes, iters = eng.heights(host, int(bound), matrix_free=(method == "naive"), lazy=(method == "lazy"))
        return host, codes, iters
    dev = torch.empty((count, NCOEFF), dtype=torch.uint8, device=f"cuda:{device}")
    _, clean = eng.sample(seed, worker, count, out=dev)
    if not clean:
        host = sample_block(p, count, seed, worker)
        codes, iters = eng.heights(host, int(bound), matrix_free=(method == "naive"), lazy=(method == "lazy"))
        return host, codes, iters
    hs, its = eng.heights(dev, int(bound), matrix_free=(method == "naive"), lazy=(method == "lazy"))
    return dev, hs.cpu().numpy(), its.cpu().numpy()


def worker_block(cfg: SearchConfig, worker: int, start: int, count: int, device: int = 0, compute=None):
    """GPU counterpart of search._worker_block: sample the block, one batched height call, summarise.

    On the engine the block never leaves the device (device_block).  `compute(p, coeffs, bound, device) -> (codes, iters)`
    replaces the engine in the CPU tests (the C oracle), with the block sampled on the host.
    """
    bound = cfg.bound if cfg.bound is not None else default_bound(cfg.n)
    if cfg.n != NVARS:
        raise DomainError(f"the GPU engine handles quartics in 4 variables; got n={cfg.n}")
    if compute is None:
        coeffs, codes, _ = device_block(cfg.p, count, cfg.rng_seed, worker, device, bound)
    else:
        coeffs = sample_block(cfg.p, count, cfg.rng_seed, worker)
        codes, _ = compute(cfg.p, coeffs, bound, device)
    return _finish_block(cfg, start, coeffs, np.asarray(codes))


def merge_results(results):
    """Merge per-worker (hist, found, best) in worker order and replay the new-maximum rule (search.py:141-153)."""
    hist, found, _ = results[0]
    found = list(found)
    for other_hist, other_found, _ in results[1:]:
        hist.merge(other_hist)
        found.extend(other_found)
    found.sort(key=lambda s: s.index)
    merged, best = [], 0
    for s in found:
        if s.height > best:
            best = s.height
            merged.append(s)
    hist.check()
    return hist, merged


def run_search(cfg: SearchConfig, devices=None, compute=None):
    """Heights of sample_count random surfaces as a histogram plus the new-maximum log (search.py:121-154).

    `parallelism` workers as in the reference; worker w runs on `devices[w % len(devices)]` (default [0]),
    concurrently when it has a device of its own.
    """
    devs = [0] if devices is None else [int(d) for d in devices]
    blocks = split_blocks(cfg.sample_count, min(cfg.parallelism, cfg.sample_count))
    results = [None] * len(blocks)
    errors = []

    def run(w):
        try:
            start, count = blocks[w]
            results[w] = worker_block(cfg, w, start, count, devs[w % len(devs)], compute)
        except Exception as exc:
            errors.append(exc)

    lanes = [[w for w in range(len(blocks)) if w % len(devs) == k] for k in range(len(devs))]
    threads = [threading.Thread(target=lambda ws=ws: [run(w) for w in ws]) for ws in lanes if ws]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return merge_results(results)


# ---- spectrum search (paper section 7) --------------------------------------------------------

def spectrum_search(p: int, block: int = 100000, rng_seed: int = 0, bound: int = 10, max_blocks: int = 1000,
                    devices=None, compute=None, want=None, progress=None, method: str = "matrix"):
    """Sample seeded blocks until every height in `want` (default 1..bound and infinity) has a witness.

    Block b uses the reference stream `default_rng([rng_seed, b])`, so any witness can be regenerated from
    (rng_seed, b, index).  One host thread per device takes the next block number, has the block sampled AND solved on its
    GPU (device_block: nothing but the height codes crosses the bus) and the blocks are retired in block order, so the result
    does not depend on the number of devices and the host does no per-sample work.
    Returns (witnesses {height code: (block, index, Quartic)}, HeightHistogram, blocks_done); height code
    0 = infinity.  `progress(blocks_done, hist, witnesses)` is called after every retired block.
    `method` = "matrix" (operator matrix built and streamed), "lazy" (the same, built only where the cap row of the first
    step does not decide) or "naive" (matrix-free iteration); same heights.
    """
    devs = [0] if devices is None else [int(d) for d in devices]
    want = set(range(0, bound + 1)) if want is None else {0 if (isinstance(h, float) and math.isinf(h)) else int(h) for h in want}
    hist = HeightHistogram(bound)
    witnesses = {}
    done = {}
    cond = threading.Condition()
    stop = threading.Event()
    errors = []
    ticket = [0]            # next block number; a consumer takes one at a time, at most 2 per device ahead of the retired front
    front = [0]

    def consume(dev):
        try:
            while not stop.is_set():
                with cond:
                    while ticket[0] - front[0] >= 2 * len(devs) and not stop.is_set():
                        cond.wait(timeout=0.1)
                    if stop.is_set() or ticket[0] >= max_blocks:
                        break
                    blk = ticket[0]
                    ticket[0] += 1
                if compute is None:
                    coeffs, codes, _ = device_block(p, block, rng_seed, blk, dev, bound, method)   # sampled and solved on the GPU
                else:
                    coeffs = sample_block(p, block, rng_seed, blk)
                    codes, _ = compute(p, coeffs, bound, dev)
                with cond:
                    done[blk] = (coeffs, np.asarray(codes))
                    cond.notify_all()
        except Exception as exc:
            errors.append(exc)
            with cond:
                cond.notify_all()

    threads = [threading.Thread(target=consume, args=(d,), daemon=True) for d in devs]
    for t in threads:
        t.start()
    nxt = 0
    while nxt < max_blocks and not want.issubset(witnesses) and not errors:
        with cond:
            while nxt not in done and not errors:
                cond.wait(timeout=0.1)
            if errors:
                break
            coeffs, codes = done.pop(nxt)
        hist.record_codes(codes)
        for h in np.unique(codes):
            h = int(h)
            if h not in witnesses:
                i = int(np.nonzero(codes == h)[0][0])
                witnesses[h] = (nxt, i, Quartic(_row(coeffs, i), p))
        nxt += 1
        with cond:
            front[0] = nxt
            cond.notify_all()
        if progress is not None:
            progress(nxt, hist, witnesses)
    stop.set()
    for t in threads:
        t.join(timeout=60)
    if errors:
        raise errors[0]
    return witnesses, hist, nxt


def spectrum_rows(witnesses) -> str:
    """Witnesses as fixture-table rows `p ; height ; poly` (k3_tables.txt format), finite heights first."""
    lines = []
    for h in sorted(witnesses, key=lambda x: (x == 0, x)):
        _, _, f = witnesses[h]
        lines.append(f"{f.modulus} ; {'inf' if h == 0 else h} ; {poly_to_text(f)}")
    return "\n".join(lines)


# ---- fixtures -------------------------------------------------------------------------------------------------

@dataclass(frozen=True)
class FixtureRow:
    line: int
    p: int
    expected: object
    f: Quartic
    text: str


@dataclass(frozen=True)
class FixtureVerdict:
    row: FixtureRow
    got: object

    @property
    def ok(self) -> bool:
        return self.got == self.row.expected


def parse_fixtures(text: str, n: int = 4):
    """Rows of `p ; height ; polynomial`, with # comments and inf (search.py:181-209)."""
    rows = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        parts = [part.strip() for part in line.split(";", 2)]
        if len(parts) != 3:
            raise ParseError(f"fixture line {lineno} needs 'p ; height ; poly'")
        try:
            p = int(parts[0])
        except ValueError:
            raise ParseError(f"fixture line {lineno}: bad prime {parts[0]!r}") from None
        if parts[1] == "inf":
            expected = INFINITE
        else:
            try:
                expected = int(parts[1])
            except ValueError:
                raise ParseError(f"fixture line {lineno}: bad height {parts[1]!r}") from None
        try:
            f = parse_poly(parts[2], n, p)
        except ParseError as exc:
            raise ParseError(f"fixture line {lineno}: {exc}") from None
        rows.append(FixtureRow(lineno, p, expected, f, parts[2]))
    return rows


def verify_fixtures(text: str, n: int = 4, primes=None, jobs: int = 1, method: str = "matrix", devices=None,
                    compute=None):
    """Recompute each fixture row's height on the GPU; verdicts in file order (search.py:219-229).

    Rows are grouped by prime and each group is one batched call.  `method` = "matrix" or "naive" as in the
    reference ("naive" = the matrix-free polynomial iteration, csrc/qfs_free.cuh); "literal" = the definitions executed
    literally (csrc/qfs_literal.cuh, rows with p <= 7 only).
    `jobs` is ignored (one batched call replaces the reference's process pool).
    """
    if method not in ("matrix", "naive", "literal", "lazy"):
        raise DomainError(f"unknown method {method!r}")
    rows = parse_fixtures(text, n)
    if primes is not None:
        keep = set(primes)
        rows = [r for r in rows if r.p in keep]
    got = [None] * len(rows)
    for p in sorted({r.p for r in rows}):
        idx = [i for i, r in enumerate(rows) if r.p == p]
        coeffs = np.stack([rows[i].f.coeffs for i in idx])
        for i in idx:
            SurfaceProblem(p, n, rows[i].f)  # the reference validates every row the same way
        if compute is None:
            codes, _ = height_batch(p, coeffs, default_bound(n), devices=devices, method=method)
        else:
            codes, _ = compute(p, coeffs, default_bound(n), 0)
        for i, c in zip(idx, codes):
            got[i] = decode_height(c)
    return [FixtureVerdict(r, g) for r, g in zip(rows, got)]


def histogram_text(hist: HeightHistogram, p: int) -> str:
    """Aligned text rendering with the 1/p^h reference column (search.py:232-242)."""
    lines = [f"{'height':>8} {'count':>10} {'fraction':>10} {'1/p^h':>10}"]
    for h in sorted(hist.counts):
        frac = hist.counts[h] / hist.total
        lines.append(f"{h:>8} {hist.counts[h]:>10} {frac:>10.5f} {1 / p**h:>10.5f}")
    if hist.infinite:
        frac = hist.infinite / hist.total
        lines.append(f"{'inf':>8} {hist.infinite:>10} {frac:>10.5f} {'':>10}")
    lines.append(f"{'total':>8} {hist.total:>10}")
    return "\n".join(lines)


def found_surfaces_text(found) -> str:
    if not found:
        return "no finite-height surfaces recorded"
    return "\n".join(f"sample {s.index}: height {s.height}: {poly_to_text(s.f)}" for s in found)
