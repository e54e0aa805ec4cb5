"""Exhaustive interleaving check of the 4-CTA multicast kernel's operand pipeline (tc_gemm.cuh, kCl = 4, NSUB = 2).

A host-side model, no GPU: is the barrier protocol itself free of deadlock, phase aliasing and smem races under
ARBITRARY skew between the four CTAs and arbitrary delay of every asynchronous signal?  (The time-slicing hang of
DESIGN.md §9 raises the question: unbounded skew is exactly what a context switch adds.)

Model — one cluster = pairs P ∈ {0, 1} × ranks r ∈ {0, 1}; STAGES ring slots; K-loop of N steps:
  * mbarrier = (phase, pending arrivals, tx-count); a phase completes when pending == 0 and tx == 0 and then pending is
    re-armed; wait(parity) passes iff the barrier's current phase parity differs from it (mbarrier.try_wait.parity).
  * producer of CTA (P, r), step i, slot s = i mod STAGES, ph = (i div STAGES) & 1:
      wait(empty[P,r][s], ph ^ 1);  if r == 0: arrive.expect_tx(full[P][s], 6 units)
      A load  → 1 unit into (P, r)'s slot, complete_tx on full[P][s]                        (cta_group::2 load)
      B multicast → 1 unit into (0, r)'s and (1, r)'s slots, complete_tx on full[0][s] and full[1][s] respectively
    every delivery is an independent in-flight event that may land at any later time.
  * MMA thread of pair P (leader CTA), step i: wait(full[P][s], ph); the reads complete; tcgen05.commit multicast →
    four independent in-flight arrivals, one on each CTA's empty[s] (count 2: both pairs' commits).
Checked in every reachable state: no deadlock; at the start of MMA step i both CTAs' slots hold step i's A and both
senders' B halves; no delivery overwrites a slot whose data the pair's MMA has not consumed yet.

Exploration: breadth-first over all interleavings up to a state budget (the full space is out of reach: every in-flight
signal commutes with every other), then random walks in which a random subset of CTAs and signal kinds is starved — only
scheduled when nothing else can move — which is the unbounded skew in question.  Two mutations show the checker can fail.

  python scripts/mc_protocol_check.py [--stages 2] [--steps 6] [--walks 20000] [--exhaustive-states 200000]
"""
import argparse
import random
import sys
from collections import deque

CTAS = [(0, 0), (0, 1), (1, 0), (1, 1)]   # (pair, rank)
FULL_TX = 6                                # 2 A units + 4 B units per pair and step


def explore(stages: int, steps: int, break_protocol: str = "", walks: int = 0, seed: int = 0,
            max_states: int = 10 ** 9):
    # state = (prod_pc[4], mma_pc[2], full[2][stages], empty[4][stages], slots, inflight)
    # prod_pc: (step, sub) with sub 0 = before the empty wait, 1 = armed, loads not issued yet
    # full barrier: (phase, pending, tx); empty barrier: (phase, pending)
    # slots[c][s] = (A version, B version from pair 0's sender, B version from pair 1's sender)
    empty_count = 1 if break_protocol == "empty_count_1" else 2
    full_tx = FULL_TX + (1 if break_protocol == "full_tx_7" else 0)
    full0 = tuple(tuple((0, 1, 0) for _ in range(stages)) for _ in range(2))
    empty0 = tuple(tuple((0, empty_count) for _ in range(stages)) for _ in range(4))
    slots0 = tuple(tuple((-1, -1, -1) for _ in range(stages)) for _ in range(4))
    init = (tuple((0, 0) for _ in range(4)), (0, 0), full0, empty0, slots0, ())
    seen = {init}
    todo = deque([init])
    n_states = 0

    def full_update(full, P, s, d_pending, d_tx):
        ph, pend, tx = full[P][s]
        pend -= d_pending
        tx += d_tx
        if pend == 0 and tx == 0:
            ph, pend = ph + 1, 1
        row = full[P][:s] + ((ph, pend, tx),) + full[P][s + 1:]
        return full[:P] + (row,) + full[P + 1:]

    def empty_arrive(empty, c, s):
        ph, pend = empty[c][s]
        pend -= 1
        if pend == 0:
            ph, pend = ph + 1, empty_count
        row = empty[c][:s] + ((ph, pend),) + empty[c][s + 1:]
        return empty[:c] + (row,) + empty[c + 1:]

    def successors(st):
        prod, mma, full, empty, slots, infl = st
        succ = []
        # ---- producers
        for c, (P, r) in enumerate(CTAS):
            i, sub = prod[c]
            if i >= steps:
                continue
            s, ph = i % stages, (i // stages) & 1
            if sub == 0:
                if (empty[c][s][0] & 1) != (ph ^ 1):          # wait(empty, ph ^ 1) passes
                    f2 = full_update(full, P, s, 1, full_tx) if r == 0 else full
                    p2 = prod[:c] + ((i, 1),) + prod[c + 1:]
                    succ.append((p2, mma, f2, empty, slots, infl))
            else:                                              # issue the A load and the B multicast
                ev = [("A", c, s, i, P)]
                ev += [("B", CTAS.index((Q, r)), s, i, P) for Q in (0, 1)]   # dest CTA, slot, version, sender pair
                p2 = prod[:c] + ((i + 1, 0),) + prod[c + 1:]
                succ.append((p2, mma, full, empty, slots, tuple(sorted(infl + tuple(ev)))))
        # ---- MMA threads
        for P in (0, 1):
            i = mma[P]
            if i >= steps:
                continue
            s, ph = i % stages, (i // stages) & 1
            if (full[P][s][0] & 1) != ph:                      # wait(full, ph) passes
                for r in (0, 1):
                    c = CTAS.index((P, r))
                    if slots[c][s] != (i, i, i):
                        return None, f"RACE: MMA of pair {P} step {i} reads slot {s} of CTA {(P, r)} = {slots[c][s]}"
                ev = tuple(("E", c, s, i, P) for c in range(4))
                m2 = mma[:P] + (i + 1,) + mma[P + 1:]
                succ.append((prod, m2, full, empty, slots, tuple(sorted(infl + ev))))
        # ---- deliveries of in-flight asynchronous events (each distinct event once)
        for k, e in enumerate(infl):
            if k > 0 and infl[k - 1] == e:
                continue
            kind, c, s, i, src = e
            rest = infl[:k] + infl[k + 1:]
            if kind == "E":
                succ.append((prod, mma, full, empty_arrive(empty, c, s), slots, rest))
                continue
            P = CTAS[c][0]
            a, b0, b1 = slots[c][s]
            old = a if kind == "A" else (b0 if src == 0 else b1)
            if old >= mma[P] and old >= 0:
                return None, (f"RACE: {kind} of step {i} overwrites step {old} in slot {s} of CTA {CTAS[c]} before "
                                  f"pair {P}'s MMA (at step {mma[P]}) consumed it")
            new = (i, b0, b1) if kind == "A" else ((a, i, b1) if src == 0 else (a, b0, i))
            row = slots[c][:s] + (new,) + slots[c][s + 1:]
            sl2 = slots[:c] + (row,) + slots[c + 1:]
            succ.append((prod, mma, full_update(full, P, s, 0, -1), empty, sl2, rest))
        done = all(p[0] >= steps for p in prod) and all(m >= steps for m in mma)
        if not succ and not done:
            return None, f"DEADLOCK: producers {prod} MMA {mma} full {full} empty {empty}"
        return succ, ""

    if walks > 0:
        # random walks with adversarial skew: in every walk a random subset of threads and event kinds is starved
        # (chosen only when nothing else is enabled), which is what a context switch does to a CTA or a signal
        rng = random.Random(seed)
        for w in range(walks):
            starve_c = {c for c in range(4) if rng.random() < 0.3}
            starve_kind = {k for k in "ABE" if rng.random() < 0.3}
            st = init
            while True:
                n_states += 1
                succ, err = successors(st)
                if err:
                    return n_states, err + f" (walk {w})"
                if not succ:
                    break

                def starved(n):
                    # which transition produced n: compare thread counters / the event that left the in-flight set
                    if n[0] != st[0]:
                        return any(n[0][c] != st[0][c] for c in starve_c)
                    if n[1] != st[1]:
                        return False
                    gone = [e for e in st[5] if st[5].count(e) > n[5].count(e)]
                    return bool(gone) and (gone[0][0] in starve_kind or gone[0][1] in starve_c)

                pref = [n for n in succ if not starved(n)]
                st = rng.choice(pref or succ)
        return n_states, ""
    while todo:
        st = todo.popleft()
        n_states += 1
        if n_states > max_states:
            return n_states, ""
        succ, err = successors(st)
        if err:
            return n_states, err
        for n in succ:
            if n not in seen:
                seen.add(n)
                todo.append(n)
    return n_states, ""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=2)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--walks", type=int, default=20000, help="random walks with adversarial starvation")
    ap.add_argument("--exhaustive-states", type=int, default=200000,
                    help="breadth-first exhaustive exploration, cut off after this many states (0 = skip)")
    a = ap.parse_args()
    bad = False
    if a.exhaustive_states > 0:
        n, err = explore(a.stages, a.steps, max_states=a.exhaustive_states)
        print(f"[protocol] breadth-first, stages={a.stages} steps={a.steps}: {n} states "
              f"({'cut off' if n > a.exhaustive_states else 'complete'}), " + (err or "no deadlock, no race"))
        bad |= bool(err)
    n, err = explore(a.stages, a.steps, walks=a.walks, seed=1)
    print(f"[protocol] {a.walks} random walks with starved CTAs / signals, stages={a.stages} steps={a.steps}: "
          f"{n} transitions, " + (err or "no deadlock, no race"))
    bad |= bool(err)
    # the checker must be able to fail: with empty[] counting one commit instead of two a producer may refill a slot
    # the other pair has not consumed
    n2, err2 = explore(a.stages, a.steps, "empty_count_1", walks=a.walks, seed=2)
    print(f"[protocol] mutation (empty[] counts one commit): " + (err2 or "NOT DETECTED"))
    n3, err3 = explore(a.stages, a.steps, "full_tx_7", walks=10, seed=3)
    print(f"[protocol] mutation (full[] expects one unit too many): " + (err3 or "NOT DETECTED"))
    return 0 if (not bad and err2 and err3) else 1


if __name__ == "__main__":
    sys.exit(main())
