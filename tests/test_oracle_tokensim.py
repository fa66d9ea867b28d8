"""P6: hit accounting (step 5.6) against an independent per-TOKEN residency model.

The model knows nothing about blocks' classes: it tracks, for every program
token, where its KV currently is (('hbm', r) / ('host', r) / None), replaying
the oracle's per-tick physical moves and fills at token granularity
(token t lives in block t // bt).  At every FETCH of a resumed program it
recomputes the classes of SPEC.md:145/165 (resume-time historical tokens:
hit / peer / host / miss) from scratch and compares with the decision."""
import pytest

import oracle
import tracegen
from tests.test_oracle_invariants import stress_cfg


class TokenSim:
    def __init__(self, bt):
        self.bt = bt
        self.where = {}      # (pid, t) -> ('hbm', r) | ('host', r)
        self.valid = {}      # pid -> number of tokens whose KV was ever written

    def classes(self, p, r):
        hit = peer = host = miss = 0
        for t in range(self.valid.get(p, 0)):
            w = self.where.get((p, t))
            if w is None:
                miss += 1
            elif w[0] == "host":
                host += 1
            elif w[1] == r:
                hit += 1
            else:
                peer += 1
        return hit, peer, host, miss

    def apply(self, moves, fills, stopped):
        bt = self.bt
        for kind, sr, si, dr, di, p, j in moves:
            for t in range(j * bt, min((j + 1) * bt, self.valid.get(p, 0))):
                if kind == oracle.ta_oracle.MOVE_DROP:
                    self.where.pop((p, t), None)
                elif kind == oracle.ta_oracle.MOVE_D2H:
                    self.where[(p, t)] = ("host", dr)
                else:                                   # P2P / H2D / D2D land in HBM of dr
                    self.where[(p, t)] = ("hbm", dr)
        for kind, r, idx, p, j, t0, t1 in fills:
            for t in range(t0, t1):
                self.where[(p, t)] = ("hbm", r)
            self.valid[p] = max(self.valid.get(p, 0), t1)
        for p in stopped:
            for t in range(self.valid.pop(p, 0)):
                self.where.pop((p, t), None)


@pytest.mark.parametrize("seed,R", [(51, 2), (52, 3), (53, 1)])
def test_hit_accounting_matches_token_model(seed, R):
    cfg = stress_cfg(seed, R=R, NB=56 if R > 1 else 80)
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    sim = TokenSim(o.bt)
    n_checked = 0
    for _ in range(300):
        before = list(o.status)
        st, dec = o.sched_step()
        # classes are computed on the residency at the start of the tick (5.6 precedes
        # 5.4; a materializing program is REASONING, so 5.3 evictions never touch it)
        for d in dec:
            if d[0] == oracle.D_FETCH and (d[7] + d[8] + d[9] + d[10]) > 0:
                assert sim.classes(d[1], d[3]) == (d[7], d[8], d[9], d[10]), d
                n_checked += 1
        stopped = [p for p in range(o.N) if o.status[p] == oracle.STOPPED and before[p] != oracle.STOPPED]
        sim.apply(o.moves, o.fills, stopped)
        for p in range(o.N):
            if o.status[p] in (oracle.PAUSED, oracle.REASONING, oracle.ACTING):
                assert sim.valid.get(p, 0) == o.c_kv[p]
        if o.next_arrival == o.N and all(s == oracle.STOPPED for s in o.status):
            break
    assert n_checked > 5
