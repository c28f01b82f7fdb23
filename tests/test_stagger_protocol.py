"""CPU model of grouped_gemm_stagger_kernel's barrier protocol (csrc/gemm.cu; one CTA view):
the TMA producer, the MMA issuer and the epilogue as coroutines over mbarrier phase
semantics (try_wait.parity(P) passes once the phase of parity P has completed), in random
interleavings.
Checks: no deadlock, every MMA reads the A/B blocks of its (tile, kb), no ring slot is
overwritten before its consumers committed, accumulators are not overwritten before the
epilogue drained them, the epilogue sees complete accumulators."""
import random


class Bar:
    def __init__(self, count):
        self.count, self.pending, self.done = count, count, 0

    def arrive(self):
        self.pending -= 1
        assert self.pending >= 0
        if self.pending == 0:
            self.done += 1
            self.pending = self.count

    def ready(self, parity):
        return (self.done & 1) != parity


def run(tiles_K, L=3, NA=5, NB=2, seed=0):
    rnd = random.Random(seed)
    fullA = [Bar(1) for _ in range(NA)]; emptyA = [Bar(1) for _ in range(NA)]
    fullB = [[Bar(1) for _ in range(NB)] for _ in range(2)]; emptyB = [[Bar(1) for _ in range(NB)] for _ in range(2)]
    tfull = [Bar(1), Bar(1)]; tempty = [Bar(1), Bar(1)]
    sA = [None] * NA; sB = [[None] * NB for _ in range(2)]
    acc = [None, None]  # (tile, h, kb_done)
    log = []

    def producer():
        seqA, seqB = 0, [0, 0]
        for t, K in enumerate(tiles_K):
            for sl in range(K + L if K > 0 else 0):
                for h in (0, 1):
                    kb = sl if h == 0 else sl - L
                    if kb < 0 or kb >= K:
                        continue
                    if h == 0:
                        a, pa = seqA % NA, (seqA // NA) & 1
                        while not emptyA[a].ready(pa ^ 1):
                            yield False
                        sA[a] = (t, kb); fullA[a].arrive(); seqA += 1
                    b, pb = seqB[h] % NB, (seqB[h] // NB) & 1
                    while not emptyB[h][b].ready(pb ^ 1):
                        yield False
                    sB[h][b] = (t, h, kb); fullB[h][b].arrive(); seqB[h] += 1
                    yield True

    def mma():
        seqA, seqB, accph = 0, [0, 0], [0, 0]
        for t, K in enumerate(tiles_K):
            if K == 0:
                for h in (0, 1):
                    while not tempty[h].ready(accph[h] ^ 1):
                        yield False
                    acc[h] = (t, h, 0); tfull[h].arrive(); accph[h] ^= 1
                continue
            seqA0 = seqA
            for sl in range(K + L):
                for h in (0, 1):
                    kb = sl if h == 0 else sl - L
                    if kb < 0 or kb >= K:
                        continue
                    if kb == 0:
                        while not tempty[h].ready(accph[h] ^ 1):
                            yield False
                        acc[h] = (t, h, 0)
                    sa = seqA0 + kb; a = sa % NA
                    if h == 0:
                        while not fullA[a].ready((sa // NA) & 1):
                            yield False
                        seqA += 1
                    b = seqB[h] % NB
                    while not fullB[h][b].ready((seqB[h] // NB) & 1):
                        yield False
                    assert sA[a] == (t, kb), ("A", sA[a], t, kb, h)
                    assert sB[h][b] == (t, h, kb), ("B", sB[h][b], t, h, kb)
                    assert acc[h][0] == t and acc[h][2] == kb, ("acc", acc[h], t, h, kb)
                    acc[h] = (t, h, kb + 1)
                    emptyB[h][b].arrive()
                    if h == 1:
                        emptyA[a].arrive()
                    if kb == K - 1:
                        tfull[h].arrive()
                    seqB[h] += 1
                    if kb == K - 1:
                        accph[h] ^= 1
                    yield True

    def epilogue():
        accph = [0, 0]
        for t, K in enumerate(tiles_K):
            for h in (0, 1):
                while not tfull[h].ready(accph[h]):
                    yield False
                accph[h] ^= 1
                assert acc[h] == (t, h, K), ("epi", acc[h], t, h, K)
                for _ in range(rnd.randint(0, 3)):
                    yield True
                log.append((t, h))
                tempty[h].arrive()
                yield True

    roles = [producer(), mma(), epilogue()]
    alive = [True] * 3
    stall = 0
    while any(alive):
        i = rnd.randrange(3)
        if not alive[i]:
            continue
        try:
            prog = next(roles[i])
            stall = 0 if prog else stall + 1
        except StopIteration:
            alive[i] = False
            stall = 0
        if stall > 100000:
            raise RuntimeError("deadlock")
    assert log == [(t, h) for t in range(len(tiles_K)) for h in (0, 1)]


def test_protocol_random_interleavings():
    rng = random.Random(1234)
    for L, NA, NB in ((3, 5, 2), (2, 4, 3), (4, 6, 2)):  # the kernel's three variants
        for seed in range(200):
            tiles = [rng.choice([0, 1, 2, 3, 4, 5, 16]) for _ in range(rng.randint(1, 5))]
            run(tiles, L=L, NA=NA, NB=NB, seed=seed)


def test_model_detects_an_undersized_a_ring():
    """NA = L: A(kb + NA) would wait on half 1's commit of A(kb), which comes L steps later."""
    import pytest

    with pytest.raises(RuntimeError, match="deadlock"):
        run([16, 16], L=3, NA=3, seed=0)
