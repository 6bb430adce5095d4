"""An independently written, set-based model of the §8(c) semantics, used only to cross-check the oracle by
brute-force enumeration.  It is deliberately structured differently from oracle/pool.py:
sets and dicts instead of state arrays, provenance instead of bytes, counters recomputed from scratch.
"""
from __future__ import annotations

INVAL, NOBLOCKS, NOHOST, HANDLE, BUSY = -1, -2, -3, -4, -5


class Fail(Exception):
    def __init__(self, status):
        self.status = status


class SetModel:
    def __init__(self, N, S, ncls=2, P=0):
        self.N, self.S, self.P = N, S, P
        self.free = set(range(N))
        self.pend = []                   # list of (cls, frozenset ids, epoch)
        self.ep = 0                      # retire / sync points so far (reading A8')
        self.back_ep = []                # epoch of each released slot in self.back
        self.own = {}                    # id -> (agent, pos)
        self.tab = {}                    # agent -> list
        self.cls = {}
        self.res = [0] * ncls
        self.clm = [0] * ncls
        self.stack = list(range(S))[::-1]
        self.pstack = list(range(S, S + P))[::-1]    # peer-tier slots (NEXT-2), ids after the host slots
        self.back = []
        self.live = {}                   # handle -> (agent, cls, pos list, slot list)
        self.dead = set()
        self.nh = 0
        self.prov = {b: b for b in range(N)}   # physical block -> original content id
        self.hprov = {}
        self.rplan = {}                  # handle -> [chunks, ticks] of an active gradual reservation
        self.rsv = {}                    # handle -> destination ids claimed so far

    def _take(self, c, n):
        unc = [max(0, self.res[x] - self.clm[x]) for x in range(len(self.res))]
        from_res = unc[c] if unc[c] < n else n
        if n > len(self.free) or n - from_res > max(0, len(self.free) - sum(unc)):
            raise Fail(NOBLOCKS)
        got = sorted(self.free)[:n]
        self.clm[c] += from_res
        self.free.difference_update(got)
        return got

    def add(self, a, c):
        self.tab[a] = []
        self.cls[a] = c

    def reserve(self, c, n):
        if sum(self.res) - self.res[c] + n > self.N:
            raise Fail(INVAL)
        self.res[c] = n

    def alloc(self, a, n):
        got = self._take(self.cls[a], n)
        for b in got:
            self.own[b] = (a, len(self.tab[a]))
            self.tab[a].append(b)
        return got

    def offload(self, a, ids):
        if not ids or len(set(ids)) < len(ids) or any(self.own.get(b, (None,))[0] != a for b in ids):
            raise Fail(INVAL)
        # whole offload to the peer tier if it fits there, else to the host tier, else refused
        tier = self.pstack if len(self.pstack) >= len(ids) else self.stack
        if len(tier) < len(ids):
            raise Fail(NOHOST)
        slots = []
        pos = []
        for b in ids:
            s = tier.pop()
            slots.append(s)
            self.hprov[s] = self.prov[b]
            p = self.own.pop(b)[1]
            pos.append(p)
            self.tab[a][p] = -1
        self.pend.append((self.cls[a], frozenset(ids), self.ep))
        self.nh += 1
        self.live[self.nh] = (a, self.cls[a], pos, slots)
        return self.nh

    def upload(self, h):
        if h not in self.live:
            raise Fail(HANDLE)
        a, c, pos, slots = self.live[h]
        mine = self.rsv.get(h, [])
        got = list(mine) + (self._take(c, len(pos) - len(mine)) if len(pos) > len(mine) else [])
        self.rsv.pop(h, None)
        self.rplan.pop(h, None)
        for p, s, b in zip(pos, slots, got):
            self.prov[b] = self.hprov[s]
            self.own[b] = (a, p)
            self.tab[a][p] = b
        self.back += slots
        self.back_ep += [self.ep] * len(slots)
        del self.live[h]
        self.dead.add(h)
        return got

    def begin(self, h, cyc):
        if h not in self.live:
            raise Fail(HANDLE)
        if cyc < 1 or h in self.rplan or self.rsv.get(h):
            raise Fail(INVAL)
        n = len(self.live[h][2])
        q, m = divmod(n, cyc)
        self.rplan[h] = [[q + 1] * m + [q] * (cyc - m), 0]
        self.rsv[h] = []

    def tick(self):
        for h in sorted(self.rplan):
            chunks, t = self.rplan[h]
            t += 1
            self.rplan[h][1] = t
            c = self.live[h][1]
            want = sum(chunks[:t]) - len(self.rsv[h])
            unc = [max(0, self.res[x] - self.clm[x]) for x in range(len(self.res))]
            room = max(0, len(self.free) - sum(unc))
            k = min(want, len(self.free), unc[c] + room)
            if k > 0:
                self.rsv[h] += self._take(c, k)

    def cancel(self, h):
        if h not in self.live:
            raise Fail(HANDLE)
        mine = self.rsv.pop(h, [])
        self.rplan.pop(h, None)
        self.free.update(mine)
        c = self.live[h][1]
        self.clm[c] = max(0, self.clm[c] - len(mine))

    def sync(self):
        self._retire(self.ep + 1)

    def retire(self, lag=1):
        if lag < 1:
            raise Fail(INVAL)
        self._retire(max(0, self.ep - (lag - 1)))

    def _retire(self, upto):
        still = []
        for c, ids, e in self.pend:
            if e < upto:
                self.free |= ids
                self.clm[c] = max(0, self.clm[c] - len(ids))
            else:
                still.append((c, ids, e))
        self.pend = still
        go = [s for s, e in zip(self.back, self.back_ep) if e < upto]
        self.stack += [s for s in go if s < self.S]
        self.pstack += [s for s in go if s >= self.S]
        keep = [(s, e) for s, e in zip(self.back, self.back_ep) if e >= upto]
        self.back = [s for s, _ in keep]
        self.back_ep = [e for _, e in keep]
        self.ep += 1

    def agent_free(self, a):
        if any(v[0] == a for v in self.live.values()):
            raise Fail(BUSY)
        mine = [b for b in self.tab[a] if b >= 0]
        for b in mine:
            del self.own[b]
        self.free.update(mine)
        c = self.cls[a]
        self.clm[c] = max(0, self.clm[c] - len(mine))
        self.tab[a] = []

    # ---- one cycle's batches (readings B1, B5).  Written as validate-then-apply: every item is checked in
    # order against the state the earlier items would leave (ownership, distinct ids, host / peer room, block room
    # under the partition rule) without touching anything, and only a fully valid batch is applied item by item.
    def _check_offloads(self, items):
        gone = set()
        room_p, room_h = len(self.pstack), len(self.stack)
        for a, ids in items:
            if not ids or len(set(ids)) < len(ids) or any(b in gone or self.own.get(b, (None,))[0] != a for b in ids):
                raise Fail(INVAL)
            if room_p >= len(ids):
                room_p -= len(ids)
            elif room_h >= len(ids):
                room_h -= len(ids)
            else:
                raise Fail(NOHOST)
            gone.update(ids)

    def _check_uploads(self, hs):
        seen = set()
        nfree, clm = len(self.free), list(self.clm)
        for h in hs:
            if h not in self.live or h in seen:
                raise Fail(HANDLE)
            seen.add(h)
            c, pos = self.live[h][1], self.live[h][2]
            n = len(pos) - len(self.rsv.get(h, []))
            if n <= 0:
                continue
            unc = [max(0, r - k) for r, k in zip(self.res, clm)]
            r = min(unc[c], n)
            if n > nfree or n - r > max(0, nfree - sum(unc)):
                raise Fail(NOBLOCKS)
            clm[c] += r
            nfree -= n

    def offload_batch(self, items):
        self._check_offloads(items)
        return [self.offload(a, ids) for a, ids in items]

    def upload_batch(self, hs):
        self._check_uploads(hs)
        return [self.upload(h) for h in hs]

    def cycle(self, hs, items):
        # uploads' status first; the offloads are checked against the pre-cycle owners, so a block this cycle's
        # uploads allocate (free or reserved now) is never an on-GPU block of the agent: INVAL (B5)
        self._check_uploads(hs)
        self._check_offloads(items)
        news = [self.upload(h) for h in hs]
        return news, [self.offload(a, ids) for a, ids in items]

    def counts(self):
        npend = sum(len(i) for _, i, _ in self.pend)
        return len(self.free), len(self.own), npend
