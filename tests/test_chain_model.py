"""CPU check of the SBS decomposition the GPU implements.

A pure-Python model of exactly what capi.cu (event planning) and sbs.cu
(speculative chain, rejection check, per-class Fisher-Yates by generation,
gather by draw number) do, compared with the reference fixtures -- including
the two engineered rejection-sampling events, which must actually reject.
"""
import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def mix(z):
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def limit(n):
    return M64 - ((M64 % n) + 1) % n


def fy_draws(s, m):
    """Swap targets and draw count K of Rng(s).shuffle over m (rng.hpp:57-64)."""
    js, k = [], 0
    for i in range(m, 1, -1):
        while True:
            k += 1
            x = mix(s + k * GAMMA)
            if x <= limit(i):
                break
        js.append((i, x % i))
    return js, k


class ModelCursor:
    def __init__(self, counts, by_class, batch, seed):
        self.counts, self.B = list(counts), batch
        self.cur = [list(v) for v in by_class]
        self.m = [len(v) for v in by_class]
        self.gen = [0] * len(by_class)
        self.batches = 0
        self.chain = seed
        self.rejections = 0
        for c in range(len(by_class)):  # ctor events, in place
            self.cur[c] = self._event(c, self.cur[c])

    def _event(self, c, perm):
        s = self.chain
        js, k = fy_draws(s, self.m[c])
        spec_k = self.m[c] - 1 if self.m[c] >= 2 else 0
        self.rejections += k - spec_k
        p = list(perm)
        for i, j in js:
            p[i - 1], p[j] = p[j], p[i - 1]
        self.chain = mix(s + (k + 1) * GAMMA)
        return p

    def next(self, n):
        keys = []
        for c, (cnt, m) in enumerate(zip(self.counts, self.m)):
            if cnt == 0 or m == 0:
                continue
            d1 = (self.batches + n) * cnt
            g = self.gen[c] + 1
            while g * m < d1:
                keys.append(((g * m) // cnt, c, g))
                g += 1
        keys.sort()
        gens = {c: {self.gen[c]: self.cur[c]} for c in range(len(self.m))}
        for _, c, g in keys:
            gens[c][g] = self._event(c, gens[c][g - 1])
        out = []
        for b in range(n):
            for c, cnt in enumerate(self.counts):
                for k in range(cnt):
                    d = (self.batches + b) * cnt + k
                    m = self.m[c]
                    out.append(gens[c][d // m][d % m])
        for c in range(len(self.m)):
            if gens[c]:
                g = max(gens[c])
                self.gen[c], self.cur[c] = g, gens[c][g]
        self.batches += n
        return out


def test_model_matches_reference_fixtures(golden):
    meta, arrays = golden
    a = arrays["sbs"]
    labels = (np.arange(50000) % 100)
    by_class = [list(range(c, 50000, 100)) for c in range(100)]
    counts = meta["sbs"]["plans"]["uniform100_512"]["counts"]
    cur = ModelCursor(counts, by_class, 512, 1234)
    got = []
    for n in (1, 4, 20):
        got += cur.next(n)
    assert got == a["c2_examples"][: len(got)].tolist()
    assert cur.rejections == 0
    del labels


def test_model_rejection_cases(golden):
    meta, arrays = golden
    a = arrays["sbs"]
    mem = a["rej_a_members"].tolist()
    for case in ("rej_a", "rej_b"):
        g = meta["sbs"][case]
        o = g["class_offsets"]
        cur = ModelCursor(g["counts"], [mem[o[c]:o[c + 1]] for c in range(3)], g["batch"], g["seed"])
        got = cur.next(3) + cur.next(7)
        assert got == a[f"{case}_examples"].tolist(), case
        assert cur.rejections >= 1, case  # the engineered rejection really happens


def test_model_skew(golden):
    meta, arrays = golden
    a = arrays["sbs"]
    g = meta["sbs"]["skew"]
    labels = a["skew_labels"].tolist()
    by_class = [[i for i, l in enumerate(labels) if l == c] for c in range(3)]
    cur = ModelCursor([8, 4, 4], by_class, 16, g["seed"])
    got = cur.next(13) + cur.next(37)
    assert got == a["skew_examples"].tolist()


def _model_plan(counts, m, gen, batches, n, chain):
    """ModelCursor.next's event enumeration + sort, and the no-rejection
    chain walk that gives each event's start state."""
    keys = []
    for c, (cnt, mm) in enumerate(zip(counts, m)):
        if cnt == 0 or mm == 0:
            continue
        d1 = (batches + n) * cnt
        g = gen[c] + 1
        while g * mm < d1:
            keys.append(((g * mm) // cnt, c, g))
            g += 1
    keys.sort()
    seeds = []
    for _, c, _ in keys:
        seeds.append(chain)
        chain = mix(chain + (m[c] if m[c] >= 2 else 1) * GAMMA)
    return keys, seeds, chain


def test_host_planner_matches_model():
    """optb_sbs_plan_call -- the C++ host planner the device path uses
    (counting sort of the events by batch, the host's chain walk) -- equals
    the Python model's sort and walk, on random class counts and sizes
    (empty, single-example and large classes) and mid-stream states.  Pure
    host code: runs without a GPU."""
    import ctypes as ct
    import paper_2105_00619_b200._lib as L
    rng = np.random.default_rng(5)
    u64 = lambda a: np.ascontiguousarray(a, np.uint64)  # noqa: E731
    p = lambda a: a.ctypes.data_as(ct.POINTER(ct.c_uint64))  # noqa: E731
    for trial in range(60):
        C = int(rng.integers(1, 40))
        counts = rng.integers(0, 9, C)
        m = rng.choice([0, 1, 2, 3, 7, 50, 500, 4099], C)
        batches = int(rng.integers(0, 300))
        # a consistent generation state: generations started by draws so far
        gen = np.array([(batches * c) // mm if mm and c else 0 for c, mm in zip(counts, m)])
        gen = np.array([g - 1 if (mm and c and (batches * c) % mm == 0 and g > 0) else g
                        for g, c, mm in zip(gen, counts, m)])
        n = int(rng.integers(1, 200))
        chain = int(rng.integers(0, 2 ** 63)) * 2 + 1
        keys, seeds, after = _model_plan(counts.tolist(), m.tolist(), gen.tolist(), batches, n, chain)
        cap = max(len(keys), 1)
        ev_c, ev_g, ev_s = (np.zeros(cap, np.uint64) for _ in range(3))
        ne, ca = ct.c_uint64(), ct.c_uint64()
        L.check(L.lib.optb_sbs_plan_call(C, p(u64(counts)), p(u64(m)), p(u64(gen)), batches, n, chain, cap,
                                         p(ev_c), p(ev_g), p(ev_s), ct.byref(ne), ct.byref(ca)))
        assert ne.value == len(keys), trial
        assert [int(x) for x in ev_c[:len(keys)]] == [k[1] for k in keys], trial
        assert [int(x) for x in ev_g[:len(keys)]] == [k[2] for k in keys], trial
        assert [int(x) for x in ev_s[:len(keys)]] == seeds, trial
        assert ca.value == after, trial


def test_reciprocal_reduction_identity():
    """The parallel Fisher-Yates reduces next_below's x % i (rng.hpp:29-35)
    as q = mulhi(x, floor((2^64-1)/i)), r = x - q*i, minus i once if r >= i
    (sbs.cu mod_below): q is floor(x/i) or one less, so this is exact.
    Checked here on edge values and random draws for every class size the
    BASELINE configs use and beyond."""
    import random
    rng = random.Random(7)
    M64 = (1 << 64) - 1

    def fast(x, i):
        q = (x * (M64 // i)) >> 64
        r = x - q * i
        assert 0 <= r < 2 * i
        return r - i if r >= i else r
    sizes = list(range(2, 2049)) + [10485, 10486, 500, 50000, (1 << 20) + 1, (1 << 31) + 11, (1 << 32) - 1]
    for i in sizes:
        edges = [0, 1, i - 1, i, M64, M64 - 1, 1 << 63, (M64 // i) * i, (M64 // i) * i - 1]
        for x in edges + [rng.getrandbits(64) for _ in range(20)]:
            assert fast(x, i) == x % i, (x, i)
