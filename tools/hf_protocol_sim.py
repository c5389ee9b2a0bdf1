"""CPU model of head_fused_kernel's mbarrier protocol (head_fused.cu): every warp role is a
generator that yields the waits the kernel makes, in the kernel's order, and performs the
same arrivals / commits.  Asynchronous completions (TMA bytes, tcgen05.commit) are modelled as
immediate.  A run that cannot make progress is a protocol deadlock; a barrier that completes a
phase twice before a waiter observed it is a parity aliasing error.  Run before a GPU test:

    python tools/hf_protocol_sim.py
"""
import itertools
import sys

RB, KDY = 4, 3


class Bar:
    def __init__(self, name, count):
        self.name, self.count, self.pending, self.phase, self.completions = name, count, 0, 0, 0

    def arrive(self, n=1):
        self.pending += n
        assert self.pending <= self.count, f"{self.name}: too many arrivals"
        if self.pending == self.count:
            self.pending = 0
            self.phase ^= 1
            self.completions += 1

    def ready(self, parity):
        return self.phase != parity


def simulate(m, KB, RA=3, verbose=False):
    NP = KB // 2
    B = {}
    mk = lambda n, c: B.setdefault(n, Bar(n, c))
    fullA = [mk(f"fullA{s}", 1) for s in range(RA)]
    emptyA = [mk(f"emptyA{s}", 1) for s in range(RA)]
    fullB = [mk(f"fullB{s}", 1) for s in range(RB)]
    emptyB = [mk(f"emptyB{s}", 1) for s in range(RB)]
    dfull = [mk(f"dfull{b}", 1) for b in range(KDY)]
    dempty = [mk(f"dempty{b}", 8) for b in range(KDY)]
    m3 = [mk(f"m3done{b}", 1) for b in range(2)]
    gfull = [mk(f"gfull{b}", 4) for b in range(2)]
    gempty = [mk(f"gempty{b}", 1) for b in range(2)]
    wfull, dwdone = mk("wfull", 1), mk("dwdone", 1)
    lfull = [mk(f"lfull{b}", 1) for b in range(2)]      # two logits buffers
    lempty = [mk(f"lempty{b}", 4) for b in range(2)]
    ownA, ownB = {}, {}
    named = {"n2": [0, 0]}               # dtanh named barrier: [arrived, generation]

    def producer(pa):
        if pa:
            wfull.arrive()
        R, full, empty, own = (RA, fullA, emptyA, ownA) if pa else (RB, fullB, emptyB, ownB)
        w = 0
        for j in range(m):
            for kb in range(KB):
                s = w % R
                yield (empty[s], ((w // R) & 1) ^ 1)
                own[s] = (j, kb, w)
                full[s].arrive()
                w += 1

    def mma_a():                          # warp 1: pass A (MMA1)
        yield (wfull, 0)
        for j in range(m):
            yield (lempty[j & 1], ((j >> 1) & 1) ^ 1)
            for kb in range(KB):
                w = j * KB + kb
                s = w % RA
                yield (fullA[s], (w // RA) & 1)
                assert ownA[s] == (j, kb, w), ("MMA1 reads wrong slot", s, ownA[s], j, kb)
                emptyA[s].arrive()
                if kb == KB - 1:
                    lfull[j & 1].arrive()

    def mma_b():                          # warp 2: pass B (MMA2 + MMA3)
        yield (wfull, 0)
        dyc = u3 = 0
        for j in range(m):
            gb = j & 1
            yield (gfull[gb], (j >> 1) & 1)
            for c in range(NP):
                for h in range(2):
                    b = dyc % KDY
                    yield (dempty[b], ((dyc // KDY) & 1) ^ 1)
                    dfull[b].arrive()
                    dyc += 1
                w = j * KB + 2 * c
                s = w % RB
                assert s % 2 == 0 and s + 1 < RB
                yield (fullB[s], (w // RB) & 1)
                yield (fullB[s + 1], ((w + 1) // RB) & 1)
                assert ownB[s] == (j, 2 * c, w) and ownB[s + 1] == (j, 2 * c + 1, w + 1)
                m3[u3 & 1].arrive()
                u3 += 1
            gempty[gb].arrive()
        dwdone.arrive()

    def loss(lw):
        for j in range(m):
            yield (lfull[j & 1], (j >> 1) & 1)
            lempty[j & 1].arrive()
            gb = j & 1
            yield (gempty[gb], ((j >> 1) & 1) ^ 1)
            gfull[gb].arrive()

    def dtanh(dw):
        dyc = u3 = 0
        for j in range(m):
            p0 = j * KB
            for c in range(NP):
                for h in range(2):
                    kb = 2 * c + h
                    b = dyc % KDY
                    wk = p0 + kb
                    yield (dfull[b], (dyc // KDY) & 1)
                    dempty[b].arrive()
                    s = wk % RB
                    yield (fullB[s], (wk // RB) & 1)
                    assert ownB[s] == (j, kb, wk), ("dtanh reads wrong slot", dw, s, ownB[s], j, kb)
                    dyc += 1
                gen = named["n2"][1]
                named["n2"][0] += 1
                if named["n2"][0] == 8:
                    named["n2"] = [0, gen + 1]
                yield ("named", gen)
                if dw == 0:
                    yield (m3[u3 & 1], (u3 >> 1) & 1)
                    s = (p0 + 2 * c) % RB
                    emptyB[s].arrive()
                    emptyB[s + 1].arrive()
                u3 += 1
        yield (dwdone, 0)

    roles = {"producerA": producer(True), "producerB": producer(False), "mmaA": mma_a(), "mmaB": mma_b()}
    for i in range(4):
        roles[f"loss{i}"] = loss(i)
    for i in range(8):
        roles[f"dtanh{i}"] = dtanh(i)
    waiting = {k: None for k in roles}
    done = set()
    steps = 0
    while len(done) < len(roles):
        progress = False
        for name, g in roles.items():
            if name in done:
                continue
            while True:
                w = waiting[name]
                if w is not None and w[0] == "poll":
                    waiting[name] = None
                    try:
                        nxt = next(g)
                    except StopIteration:
                        done.add(name)
                        progress = True
                        break
                    if nxt[0] == "poll" and not nxt[1]:
                        waiting[name] = nxt
                        break                     # polled, nothing ready: yield the round
                    waiting[name] = nxt
                    progress = True
                    steps += 1
                    continue
                if w is not None:
                    if w[0] == "named":
                        if named["n2"][1] <= w[1]:
                            break
                    elif not w[0].ready(w[1]):
                        break
                try:
                    waiting[name] = next(g)
                    progress = True
                    steps += 1
                except StopIteration:
                    done.add(name)
                    progress = True
                    break
        if not progress:
            blocked = {k: (v[0].name if v and not isinstance(v[0], str) else (v[0] if v else None),
                           v[1] if v else None)
                       for k, v in waiting.items() if k not in done}
            raise RuntimeError(f"deadlock m={m} KB={KB}: {blocked}")
    return steps


if __name__ == "__main__":
    for KB, m, RA in itertools.product((2, 4, 8), (1, 2, 3, 4, 7, 8), (3, 4, 5)):
        simulate(m, KB, RA)
    print("protocol ok for KB in {2,4,8}, m in {1,2,3,4,7,8}, pass-A ring RA in {3,4,5}")
    sys.exit(0)
