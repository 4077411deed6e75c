"""The peer combine's two-slot protocol, modelled on the host: N ranks, each a
thread running steps with random delays, publish their per-step values into slot (step mod 2)
of every rank's inbox -- values first, then the sequence number step + 1 -- and take the max
once all N entries of the slot carry it.  Every rank must obtain the true max of every step
(no entry overwritten before it was read, no stale entry accepted), for any interleaving --
the property the CUDA ctrl kernel relies on (it adds the system-scope fences the host model
gets from the GIL).  Not a GPU test: it checks the protocol, not the kernel."""
import random
import threading

import pytest


def run(nranks: int, steps: int, seed: int):
    W = 2  # slots
    inbox = [[[(0, 0)] * nranks for _ in range(W)] for _ in range(nranks)]  # [owner][slot][rank]
    lock = threading.Lock()  # one entry = (value, seq) written atomically, like the fenced pair
    got = [[None] * steps for _ in range(nranks)]
    truth = [[random.Random(seed * 1000 + r * 7 + s).random() for r in range(nranks)]
             for s in range(steps)]

    def rank(r):
        rng = random.Random(seed + r)
        for s in range(steps):
            slot, seq = s % W, s + 1
            for o in range(nranks):  # publish to every inbox
                with lock:
                    inbox[o][slot][r] = (truth[s][r], seq)
                if rng.random() < 0.3:
                    threading.Event().wait(rng.random() * 1e-4)
            while True:  # wait for all entries of this slot
                with lock:
                    row = list(inbox[r][slot])
                if all(q == seq for _, q in row):
                    break
            got[r][s] = max(v for v, _ in row)
            if rng.random() < 0.2:
                threading.Event().wait(rng.random() * 1e-4)

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
        assert not t.is_alive(), "deadlock"
    for s in range(steps):
        m = max(truth[s])
        for r in range(nranks):
            assert got[r][s] == m, (r, s)


@pytest.mark.parametrize("nranks,seed", [(2, 1), (3, 2), (8, 3)])
def test_two_slot_combine_is_exact_under_any_interleaving(nranks, seed):
    run(nranks, 200, seed)
