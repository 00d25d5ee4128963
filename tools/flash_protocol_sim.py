"""Randomised simulation of the attn_flash.cu forward synchronisation protocol
(mbarrier parity waits, tcgen05.commit arrivals, TMA completions) to find
deadlocks and ordering violations on the CPU. Usage:
    python tools/flash_protocol_sim.py [trials]
Models: loader thread, MMA thread, 2 softmax "threads" (the two key halves of
a row; each stands for a warp group), in-order tensor pipe with random
latencies, TMA with random latencies."""
import random
import sys


class Bar:
    def __init__(self, count, name):
        self.count, self.name = count, name
        self.phase = 0          # completed phases
        self.pending = 0        # arrivals in the current phase
        self.tx = 0

    def arrive(self):
        self.pending += 1
        self._check()

    def expect(self, n):
        self.tx += n
        self.pending += 1
        self._check_noarrive = True

    def complete_tx(self, n):
        self.tx -= n
        self._check()

    def _check(self):
        if self.pending >= self.count and self.tx == 0:
            self.pending = 0
            self.phase += 1

    def test(self, parity):
        # try_wait.parity: true iff the current (in-progress) phase parity != parity
        return (self.phase & 1) != parity


class Sim:
    def __init__(self, probs, seed):
        self.rng = random.Random(seed)
        self.t = 0
        self.events = []  # (time, fn)
        self.probs = probs
        B = lambda c, n: Bar(c, n)  # noqa: E731
        self.bQ, self.bV = B(1, "Q"), B(1, "V")
        self.bK = [B(1, "K0"), B(1, "K1")]
        self.bS = [B(1, f"S{i}") for i in range(3)]
        self.bP = [B(2, f"P{i}") for i in range(3)]
        self.bO = B(1, "O")
        self.bO2 = [B(1, "O20"), B(1, "O21")]
        self.pipe_free = 0     # tensor pipe: in order
        self.last_done = 0
        self.log = []
        # TMEM buffer state for hazard checks
        self.buf_owner = [None, None, None]

    def later(self, dt, fn):
        self.events.append((self.t + dt, fn))

    def tma(self, bar, nbytes=1):
        # mbarrier.arrive.expect_tx: one arrival plus nbytes of pending transactions
        bar.tx += nbytes
        bar.pending += 1
        self.later(self.rng.randint(5, 60), lambda: bar.complete_tx(nbytes))

    def mma(self, name):
        start = max(self.t, self.pipe_free)
        dur = self.rng.randint(3, 20)
        self.pipe_free = start + dur
        done = self.pipe_free + self.rng.randint(0, 10)
        done = max(done, self.last_done)  # completion in order
        self.last_done = done
        self.log.append((self.t, "issue", name))
        return done

    def commit(self, bar):
        at = max(self.last_done, self.t)
        self.events.append((at + 1, lambda: bar.arrive()))


def run(seed, probs):
    s = Sim(probs, seed)
    ncount = [p for p in probs]

    def loader():
        cs = [0, 0, 0]
        co = 0
        for n in ncount:
            if co > 0:
                yield (s.bO, (co - 1) & 1)
            s.tma(s.bQ)
            s.tma(s.bK[0])
            if n > 1:
                s.tma(s.bK[1])
            s.tma(s.bV)
            for j in range(n):
                if j + 2 < n:
                    yield (s.bS[j % 3], (cs[j % 3] + j // 3) & 1)
                    s.tma(s.bK[j & 1])
                if j + 1 < n:
                    yield (s.bO, (co + j) & 1)
                    s.tma(s.bV)
            for r in range(3):
                cs[r] += (n - r + 2) // 3
            co += n
        if co > 0:
            yield (s.bO, (co - 1) & 1)

    def mma():
        nq = 0
        nk = [0, 0]
        nv = 0
        np_ = [0, 0, 0]
        co = 0
        for n in ncount:
            yield (s.bQ, nq & 1)
            nq += 1
            yield ("delay", 5)  # Q conversion

            def issue_s(j):
                nonlocal nk
                yield (s.bK[j & 1], nk[j & 1] & 1)
                nk[j & 1] += 1
                s.mma(f"S{j}")
                s.commit(s.bS[j % 3])

            yield from issue_s(0)
            if n > 1:
                yield from issue_s(1)
            for j in range(n):
                yield (s.bV, nv & 1)
                nv += 1
                yield ("delay", 3)  # V conversion
                yield (s.bP[j % 3], np_[j % 3] & 1)
                np_[j % 3] += 1
                s.mma(f"PV{j}")
                s.commit(s.bO)
                s.commit(s.bO2[(co + j) & 1])
                if j + 2 < n:
                    if j >= 1:
                        k = co + j - 1
                        yield (s.bO2[k & 1], (k >> 1) & 1)
                    yield from issue_s(j + 2)
            co += n

    def softmax(kh):
        ns = [0, 0, 0]
        co = 0
        for n in ncount:
            for j in range(n):
                yield (s.bS[j % 3], ns[j % 3] & 1)
                ns[j % 3] += 1
                yield ("delay", s.rng.randint(5, 40))
                yield ("sync", j)
                if j > 0 and s.rng.random() < 0.3:
                    k = co + j - 1
                    yield (s.bO2[k & 1], (k >> 1) & 1)
                s.bP[j % 3].arrive()
            k = co + n - 1
            yield (s.bO2[k & 1], (k >> 1) & 1)
            yield ("sync", -1)
            yield ("sync", -2)
            co += n

    threads = {"loader": loader(), "mma": mma(), "sm0": softmax(0), "sm1": softmax(1)}
    waiting = {k: None for k in threads}
    sync_wait = {}
    done = set()
    for step in range(200000):
        progressed = False
        for name, th in threads.items():
            if name in done:
                continue
            w = waiting[name]
            if w is not None:
                if w[0] == "delay":
                    if s.t < w[1]:
                        continue
                elif w[0] == "sync":
                    continue
                elif not w[0].test(w[1]):
                    continue
            try:
                nxt = next(th)
            except StopIteration:
                done.add(name)
                progressed = True
                continue
            progressed = True
            if nxt[0] == "delay":
                waiting[name] = ("delay", s.t + nxt[1])
            elif nxt[0] == "sync":
                waiting[name] = ("sync", nxt[1])
                sync_wait[name] = nxt[1]
                if sync_wait.get("sm0") is not None and sync_wait.get("sm1") is not None:
                    waiting["sm0"] = waiting["sm1"] = None
                    sync_wait["sm0"] = sync_wait["sm1"] = None
            else:
                waiting[name] = nxt
        if len(done) == 4:
            return None
        if not progressed:
            # advance time to the next event
            if s.events:
                s.events.sort(key=lambda e: e[0])
                tnext = s.events[0][0]
                s.t = max(s.t + 1, tnext)
                while s.events and s.events[0][0] <= s.t:
                    _, fn = s.events.pop(0)
                    fn()
            else:
                s.t += 1
                if all(w is not None and w[0] not in ("delay",) for n2, w in waiting.items()
                       if n2 not in done):
                    return {n2: (w[0].name if hasattr(w[0], "name") else w[0], w[1])
                            for n2, w in waiting.items() if n2 not in done}
        else:
            while s.events and s.events[0][0] <= s.t:
                s.events.sort(key=lambda e: e[0])
                _, fn = s.events.pop(0)
                fn()
    return "timeout"


if __name__ == "__main__":
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    bad = 0
    for seed in range(trials):
        rng = random.Random(seed)
        probs = [rng.choice([1, 2, 3, 4, 5, 6, 8]) for _ in range(rng.randint(1, 4))]
        r = run(seed, probs)
        if r is not None:
            bad += 1
            if bad <= 5:
                print("seed", seed, "probs", probs, "stuck:", r)
    print(f"{bad} / {trials} runs stuck")
