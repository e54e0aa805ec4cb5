"""Host-side model of the 4-CTA multicast kernel's operand pipeline (scripts/mc_protocol_check.py; tc_gemm.cuh kCl = 4):
the barrier protocol must survive arbitrary skew between the CTAs and arbitrarily late asynchronous signals, and the
checker must catch a wrong arrival count or a wrong tx-count."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
import mc_protocol_check as M   # noqa: E402


def test_protocol_has_no_deadlock_or_race_under_random_starvation():
    for stages, steps in [(2, 6), (4, 10)]:
        _, err = M.explore(stages, steps, walks=300, seed=11)
        assert err == "", err
    n, err = M.explore(2, 4, max_states=20000)      # a breadth-first prefix of the full interleaving space
    assert err == "" and n > 10000


def test_checker_catches_seeded_protocol_bugs():
    _, err = M.explore(2, 6, "empty_count_1", walks=300, seed=12)
    assert err.startswith("RACE"), err
    _, err = M.explore(2, 6, "full_tx_7", walks=5, seed=13)
    assert err.startswith("DEADLOCK"), err
