"""Golden W1 (tests/golden/w1.json): a hand-computed two-tick example covering
restore-elsewhere, host fetch, decayed-ACTING eviction to host and drop, P2P
and H2D fetch."""
import json
import os

import oracle
from tests.helpers import base_cfg, flat_trace, set_program

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "w1.json")
ST = {"PAUSED": oracle.PAUSED, "REASONING": oracle.REASONING, "ACTING": oracle.ACTING}
DK = {"PAUSE": oracle.D_PAUSE, "RESTORE": oracle.D_RESTORE, "EVICT": oracle.D_EVICT,
      "FETCH": oracle.D_FETCH, "STALL": oracle.D_STALL, "COMPACT": oracle.D_COMPACT}
MK = {"D2H": 1, "P2P": 2, "H2D": 3, "D2D": 4, "DROP": 5}


def load_w1():
    g = json.load(open(GOLDEN))
    cfg = base_cfg(**g["config"])
    n = len(g["programs"])
    tr = flat_trace(n, **g["trace"])
    o = oracle.Oracle(cfg, tr)
    for pr in g["programs"]:
        set_program(o, pr["p"], ST[pr["status"]],
                    oracle.PHASE_A if pr["phase"] == "A" else oracle.PHASE_R, pr["c"],
                    placement=pr["placement"], home=pr["home"],
                    acting_since=pr.get("acting_since", 0), tool_return=pr.get("tool_return"),
                    paused_since=pr.get("paused_since", 0), satisfied=pr.get("satisfied", 0),
                    hbm=pr.get("hbm", ()), host=pr.get("host", ()))
    o.tick = g["start_tick"]
    o.next_arrival = n
    return g, o


def test_w1_oracle():
    g, o = load_w1()
    o.check_invariants()
    for tk in g["ticks"]:
        st, dec = o.sched_step()
        assert st == oracle.OK
        assert o.L == tk["L_after_restore"]
        want = [tuple([DK[d[0]]] + d[1:]) for d in tk["decisions"]]
        assert dec == want, (tk["tick"], dec)
        moves = [(m[0], m[1], m[2], m[3], m[4]) for m in o.moves]
        assert moves == [tuple([MK[m[0]]] + m[1:]) for m in tk["moves"]]
        o.check_invariants()
    es = g["end_state"]
    for p, row in es["loc"].items():
        p = int(p)
        want = []
        for e in row:
            want.append(oracle.NONE if e == "N" else
                        (int(e[1:]) if e[0] == "H" else oracle.HOST_BIT | int(e[1:])))
        assert list(o.loc[p][:len(want)]) == want, p
    assert o.home == es["home"]
    assert o.status == [ST[s] for s in es["status"]]
    for r, free in es["hbm_free"].items():
        assert [b for b in range(o.NB) if o.hbm_free[int(r)][b]] == free
    for r, free in es["host_free"].items():
        assert [s for s in range(o.NH) if o.host_free[int(r)][s]] == free
