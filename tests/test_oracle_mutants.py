"""Mutation check of the hand pins (VERDICT r1, next-round item 1 "done when"):
each plausible mistake in a definitional rule of the oracle -- compaction finger
order, eviction group order, host-slot order, tail-first eviction, the ceil in the
tool-call start time, the engine busy time -- is applied to an in-memory copy of
oracle/ta_oracle.py, and at least one hand-computed test of
tests/test_oracle_handpins.py must then fail."""
import types

import pytest

import oracle
from tests import test_oracle_handpins as H

SRC = open(oracle.ta_oracle.__file__).read()

MUTANTS = {
    "compaction stops one pair early": (
        "if lo >= self.NB or hi < 0 or lo > hi:",
        "if lo >= self.NB or hi < 0 or lo + 1 >= hi:"),
    "compaction moves lowest used to highest free": (
        "            p, j = self.owner_hbm[r][hi]\n            self.loc[p][j] = lo",
        "            lo, hi = hi, lo\n            p, j = self.owner_hbm[r][hi]\n            self.loc[p][j] = lo"),
    "group 0 in forward restore order": (
        "key=lambda p: self.restore_key(p, nb[p]), reverse=True)",
        "key=lambda p: self.restore_key(p, nb[p]), reverse=False)"),
    "group 2 before group 1": ("return g0 + g1 + g2", "return g0 + g2 + g1"),
    "group 1 by slot, not contribution": (
        "g1 = sorted([p for p in E if self.status[p] == ACTING and self.placement[p] != r],\n"
        "                    key=lambda p: (contrib[p], p))",
        "g1 = sorted([p for p in E if self.status[p] == ACTING and self.placement[p] != r],\n"
        "                    key=lambda p: p)"),
    "head-first eviction": ("for j in sorted(hbm_js, reverse=True)[:take]:", "for j in sorted(hbm_js)[:take]:"),
    "highest free host slot first": (
        "while hslot < self.NH and not self.host_free[r][hslot]:\n                    hslot += 1\n"
        "                if hslot < self.NH:\n                    self.host_free[r][hslot] = 0\n"
        "                    self.owner_host[r][hslot] = (p, j)\n"
        "                    row[j] = HOST_BIT | hslot",
        "while hslot < self.NH and not self.host_free[r][self.NH - 1 - hslot]:\n                    hslot += 1\n"
        "                if hslot < self.NH:\n                    self.host_free[r][self.NH - 1 - hslot] = 0\n"
        "                    self.owner_host[r][self.NH - 1 - hslot] = (p, j)\n"
        "                    row[j] = HOST_BIT | (self.NH - 1 - hslot)"),
    "floor in the tool-call start": ("ceil_div(left * 1000, self.rate)", "(left * 1000) // self.rate"),
    "engine busy time ignored": ("self.acting_since[p] = T - self.dt + busy + took",
                                 "self.acting_since[p] = T - self.dt + took"),
}

HAND_TESTS = [getattr(H, n) for n in dir(H) if n.startswith("test_")]


def _mutant_module(a, b):
    assert SRC.count(a) == 1, "mutation anchor must be unique in oracle/ta_oracle.py"
    m = types.ModuleType("ta_oracle_mutant")
    exec(compile(SRC.replace(a, b), "ta_oracle_mutant.py", "exec"), m.__dict__)
    return m


def test_hand_pins_pass_on_the_oracle():
    for t in HAND_TESTS:
        t()


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_each_mutant_fails_a_hand_pin(name, monkeypatch):
    m = _mutant_module(*MUTANTS[name])
    monkeypatch.setattr(oracle, "Oracle", m.Oracle)
    failed = []
    for t in HAND_TESTS:
        try:
            t()
        except Exception:             # a wrong value or a broken state
            failed.append(t.__name__)
    assert failed, f"mutant '{name}' survives every hand pin"
