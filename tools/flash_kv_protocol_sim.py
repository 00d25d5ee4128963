"""Randomised simulation of the synchronisation protocol of the reworked
flash dK/dV kernel (attn_flash.cu, attn_bwd_kv_flash_kernel): TMA thread, MMA
thread, an in-order tensor pipe with random latencies, TMA loads with random
latencies and NC compute groups (each stands for a set of compute warps; the
per-step named barrier among the warps sharing TMEM lanes is modelled as a
barrier among the groups). Steps are numbered globally over a CTA's
problems, as in the kernel. Checks: no deadlock; every parity wait is for the
phase the waiter means (never a phase that is two or more behind the
barrier); no read of a shared-memory stage, of K / V, of a TMEM S / P~
buffer or of the dV / dK accumulators after it was overwritten for a later
step / problem, and no overwrite before the last reader of the old content.
Usage: python tools/flash_kv_protocol_sim.py [trials]"""
import random
import sys

KST = 4  # query stages


class Bar:
    def __init__(self, count):
        self.count, self.arr, self.ph = count, 0, 0

    def arrive(self):
        self.arr += 1
        if self.arr == self.count:
            self.arr, self.ph = 0, self.ph + 1

    def ready(self, idx, who):
        # waiting for completion number idx (0-based) with try_wait.parity(idx & 1)
        assert self.ph <= idx + 1, f"{who}: parity alias (phase {self.ph}, wants completion {idx})"
        return self.ph >= idx + 1


def simulate(seed):
    R = random.Random(seed)
    nprob = R.randint(1, 7)
    steps = [R.randint(1, 5) for _ in range(nprob)]
    NC = R.choice([1, 2, 3])
    bKV, bQ = Bar(1), [Bar(1) for _ in range(KST)]
    bSD, bPD = [Bar(1) for _ in range(2)], [Bar(NC) for _ in range(2)]
    bM = [Bar(1) for _ in range(KST)]
    # shared state: who owns what
    st = dict(stage=[None] * KST, kv=None, tbuf=[None, None], pbuf=[None, None], acc=None,
              acc_read=set(), s_read={}, events=[])
    pipe, tma = [], []  # in-flight ops: (ready_time, fn)
    now = [0]
    first_k = []
    k = 0
    for n in steps:
        first_k.append(k)
        k += n
    prob_of = {}
    for p, n in enumerate(steps):
        for j in range(n):
            prob_of[first_k[p] + j] = p

    def tma_agent():
        k, klast = 0, -1
        for p, n in enumerate(steps):
            for j in range(n):
                s = k % KST
                if k >= KST:
                    while not bM[s].ready((k - KST) // KST, "tma bM"):
                        yield
                # stage s is overwritten: its last readers (S and grads of k - KST) done
                old = st["stage"][s]
                assert old is None or (isinstance(old, int) and old in st["gdone"]), \
                    f"stage {s} overwritten under step {old}"
                st["stage"][s] = ("loading", k)
                t = now[0] + R.randint(1, 40)

                def land(s=s, k=k):
                    st["stage"][s] = k
                    bQ[s].arrive()
                tma.append((t, land))
                if j == 0:
                    if klast >= 0:
                        while not bSD[klast & 1].ready(klast >> 1, "tma bSD"):
                            yield
                    # K, V overwritten: every S of earlier problems executed
                    assert all(kk in st["sdone"] for kk in range(k)), "K/V overwritten under an S MMA"
                    st["kv"] = ("loading", p)
                    t = now[0] + R.randint(1, 60)

                    def land_kv(p=p):
                        st["kv"] = p
                        bKV.arrive()
                    tma.append((t, land_kv))
                k += 1
                yield
            klast = k - 1

    def mma_agent():
        k, np_ = 0, 0
        for p, n in enumerate(steps):
            while not bKV.ready(np_, "mma bKV"):
                yield
            np_ += 1
            for j in range(n + 1):
                if j < n:
                    kk = k + j
                    while not bQ[kk % KST].ready(kk // KST, "mma bQ"):
                        yield
                    if kk >= 2:
                        while not bM[(kk - 2) % KST].ready((kk - 2) // KST, "mma bM"):
                            yield

                    def do_s(kk=kk, p=p):
                        assert st["kv"] == p, f"S({kk}) reads K/V of {st['kv']}, wants problem {p}"
                        assert st["stage"][kk % KST] == kk, f"S({kk}) reads stage holding {st['stage'][kk % KST]}"
                        b = kk & 1
                        old = st["tbuf"][b]
                        assert old is None or (old[0] == "P" and old[1] in st["gdone"]), \
                            f"S({kk}) overwrites buffer holding {old} before its grads"
                        st["tbuf"][b] = ("S", kk)
                        st["sdone"].add(kk)
                    pipe.append(("op", do_s))
                    pipe.append(("commit", bSD[kk & 1]))
                if j >= 1:
                    kk = k + j - 1
                    while not bPD[kk & 1].ready(kk >> 1, "mma bPD"):
                        yield

                    def do_g(kk=kk, p=p, first=(j == 1)):
                        b = kk & 1
                        assert st["tbuf"][b] == ("P", kk), f"grads({kk}) read buffer holding {st['tbuf'][b]}"
                        assert st["stage"][kk % KST] == kk, f"grads({kk}) reads stage holding {st['stage'][kk % KST]}"
                        if first:
                            assert st["acc"] is None or st["acc"] in st["acc_read"], "dV/dK overwritten before the epilogue read"
                            st["acc"] = p
                        else:
                            assert st["acc"] == p
                        st["gdone"].add(kk)
                    pipe.append(("op", do_g))
                    pipe.append(("commit", bM[kk % KST]))
                yield
            k += n

    def compute_agent(c, bar_state):
        k = 0
        for p, n in enumerate(steps):
            for j in range(n):
                kk = k + j
                while not bSD[kk & 1].ready(kk >> 1, f"cmp{c} bSD"):
                    yield
                for _ in range(R.randint(0, 4)):  # warps run at different speeds
                    yield
                assert st["tbuf"][kk & 1] == ("S", kk), f"cmp{c} reads S buffer holding {st['tbuf'][kk & 1]}"
                assert st["stage"][kk % KST] == kk, f"cmp{c} reads stats of stage holding {st['stage'][kk % KST]}"
                st["sread"][kk] = st["sread"].get(kk, 0) + 1
                # named barrier: every group has read S before any writes P~ over it
                bar_state[kk] = bar_state.get(kk, 0) + 1
                while bar_state[kk] < NC:
                    yield
                yield
                # each group writes its P~ / dS columns over S columns every group reads
                assert st["sread"][kk] == NC, f"cmp{c} writes P~({kk}) before every group read S({kk})"
                st["pwrites"][kk] = st["pwrites"].get(kk, 0) + 1
                if st["pwrites"][kk] == NC:
                    st["tbuf"][kk & 1] = ("P", kk)
                bPD[kk & 1].arrive()
                yield
            kl = k + n - 1
            while not bM[kl % KST].ready(kl // KST, f"cmp{c} bM"):
                yield
            assert st["acc"] == p and kl in st["gdone"], "epilogue reads an accumulator not complete"
            st["acc_reads"][p] = st["acc_reads"].get(p, 0) + 1
            if st["acc_reads"][p] == NC:
                st["acc_read"].add(p)
            yield
            k += n

    st["sdone"], st["gdone"], st["acc_reads"], st["sread"], st["pwrites"] = set(), set(), {}, {}, {}
    bar_state = {}
    agents = [tma_agent(), mma_agent()] + [compute_agent(c, bar_state) for c in range(NC)]
    alive = list(agents)
    busy_until = [0]
    idle = 0
    while alive or pipe or tma:
        now[0] += 1
        # async completions
        for item in sorted([x for x in tma if x[0] <= now[0]], key=lambda x: x[0]):
            tma.remove(item)
            item[1]()
        if pipe and now[0] >= busy_until[0]:
            kind, x = pipe.pop(0)
            if kind == "op":
                x()
                busy_until[0] = now[0] + R.randint(1, 12)
            else:
                x.arrive()  # commit: every earlier op of the in-order pipe has executed
        progressed = False
        for a in R.sample(alive, len(alive)):
            try:
                next(a)
                progressed = True
            except StopIteration:
                alive.remove(a)
        idle = 0 if (progressed or pipe or tma) else idle + 1
        assert now[0] < 200000 and idle < 2000, f"deadlock (seed {seed})"
    assert st["gdone"] == set(range(sum(steps))), "not every step finished"
    return sum(steps)


if __name__ == "__main__":
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    tot = 0
    for t in range(trials):
        tot += simulate(t)
    print(f"{trials} random schedules, {tot} steps: no deadlock, alias or hazard")
