"""Run oracle and GPU side by side, comparing full state after every tick; print the
first divergence with context (developer tool, GPU box)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import tracegen  # noqa: E402
from paper_2602_13692_b200 import Pool  # noqa: E402
from tests.gpu_compare import compare_state, dec_tuples  # noqa: E402


def main():
    name = sys.argv[1]
    over = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    ticks = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    cfg = tracegen.get_config(name, **over)
    tr = tracegen.make_trace(cfg)
    o = oracle.Oracle(cfg, tr)
    pool = Pool(cfg, tr.n_slots, max_turns=tr.total_turns)
    pool.load_trace(tr)
    for k in range(ticks):
        _, want = o.sched_step()
        st, got = pool.step()
        g = pool.debug_download()
        fp = o.fp
        for f in ("nb", "n_hbm", "contrib"):
            a = np.array(fp[f] if f != "contrib" else o.contrib, np.uint32)
            live = np.array(o.status) != oracle.UNARRIVED
            if not np.array_equal(a[live], g[f][live]):
                bad = np.nonzero((a != g[f]) & live)[0][:10]
                print(f"tick {k}: derived {f} differs at {bad}: oracle {a[bad]} gpu {g[f][bad]}")
        got = dec_tuples(got)
        if got != want:
            print(f"tick {k}: decisions differ ({len(want)} vs {len(got)})")
            for i, (x, y) in enumerate(zip(want, got)):
                if x != y:
                    print("  first", i, "oracle", x, "gpu", y)
                    break
        try:
            compare_state(o, g, where=f"tick {k}")
        except AssertionError as e:
            print("STATE:", e)
            from tests.gpu_compare import oracle_arrays
            a = oracle_arrays(o)
            NBW = -(-o.NB // 32)
            fa = np.unpackbits(a["hbm_free"].view(np.uint8), bitorder="little")
            fg = np.unpackbits(g["hbm_free"].view(np.uint8), bitorder="little")
            diff = np.nonzero(fa != fg)[0]
            print("n differing free bits", diff.size)
            for x in diff[:12]:
                r, b = divmod(int(x), NBW * 32)
                ow = o.owner_hbm[r][b] if b < o.NB else None
                og = int(g["owner_hbm"][r * o.NB + b]) if b < o.NB else -1
                print(f"  r={r} b={b} oracle_free={fa[x]} gpu_free={fg[x]} oracle_owner={ow} "
                      f"gpu_owner=({og // o.MAXB},{og % o.MAXB})")
                if ow:
                    p = ow[0]
                    print("    oracle p", p, "status", o.status[p], "home", o.home[p], "c", o.c[p],
                          "loc", list(o.loc[p][:o.nb_of(p)])[:12])
                    print("    gpu    p", p, "status", g["status"][p], "home", g["home"][p], "c", g["c"][p],
                          "loc", [int(v) for v in g["loc"][p][:o.nb_of(p)]][:12])
            st = pool.stats()
            print("stats gpu", {k2: v for k2, v in st.items() if k2 in o.stats and st[k2] != o.stats[k2]},
                  "oracle", {k2: o.stats[k2] for k2 in o.stats if k2 in st and st[k2] != o.stats[k2]})
            return
        bad, seen = pool.verify_content()
        print(f"tick {k}: ok  decisions={len(got)} verify bad={bad} seen={seen}")
        if got != want:
            return


if __name__ == "__main__":
    main()
