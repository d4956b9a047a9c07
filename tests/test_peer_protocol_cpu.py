"""Host model of the peer-mailbox protocol of the multi-GPU CGS2 (SURVEY.md
8(f2); csrc/cgs_fused.cu peer_exchange, internal.h PeerArgs).

P ranks x nb CTAs are threads.  Reduction rs (1, 2, ... as counted by every
rank): each CTA sends, to every rank q, its columns' values for slot
[rs & 1][rank] of q's mailbox followed by one arrival on q's counter
[rs & 1] (data before arrival per destination: the kernel's fence.sc.sys
before its red.release.sys).  Deliveries to different destinations are
independent and delayed at random (NVLink reorders across destinations); a
rank then waits until its own counter [rs & 1] holds ((rs + 1) // 2) * P * nb
arrivals and sums the P slots in rank order.  The sums every rank reads must
be exactly the values of that reduction: no overwrite by a fast rank's
next-but-one reduction, no arrival of reduction rs + 1 counted for rs -- the
argument DESIGN.md 9 makes for two parity banks and per-parity counters.  A
single counter (target rs * P * nb) fails the same adversarial schedule,
which shows the model can see the hazard.  CPU only.
"""
import random
import threading
import time


def run_protocol(P, nb, R, ncols, seed, per_parity=True, slow=None):
    """slow = (src, dst, rs, seconds): src's delivery to dst at reduction rs is late."""
    rng = random.Random(seed)
    mbox = [[[[None] * ncols for _ in range(P)] for _ in range(2)] for _ in range(P)]
    ctr = [[0, 0] for _ in range(P)]
    lock = threading.Lock()
    errors, timers = [], []
    barrier = [threading.Barrier(nb) for _ in range(P)]

    def value(rank, rs, j):
        return rank * 1000003 + rs * 1009 + j

    def deliver(q, rank, rs, cols, par):
        for j in cols:
            mbox[q][rs & 1][rank][j] = value(rank, rs, j)
        with lock:
            ctr[q][par] += 1

    def cta(rank, b):
        for rs in range(1, R + 1):
            par = rs & 1 if per_parity else 0
            cols = list(range(b, ncols, nb))  # the CTA's columns (warp per column in the kernel)
            for q in range(P):
                with lock:
                    d = rng.random() * 2e-3
                if slow and (rank, q, rs) == slow[:3]:
                    d = slow[3]
                t = threading.Timer(d, deliver, args=(q, rank, rs, cols, par))
                timers.append(t)
                t.start()
            target = ((rs + 1) // 2 if per_parity else rs) * P * nb
            t0 = time.time()
            while True:
                with lock:
                    if ctr[rank][par] >= target:
                        break
                if time.time() - t0 > 3:
                    errors.append(("timeout", rank, rs))
                    return
                time.sleep(2e-5)
            for j in range(ncols):
                got = [mbox[rank][rs & 1][q][j] for q in range(P)]
                if got != [value(q, rs, j) for q in range(P)]:
                    errors.append(("stale", rank, b, rs, j))
                    return
            # the kernel's next reduction follows a rank-local grid barrier
            barrier[rank].wait()

    th = [threading.Thread(target=cta, args=(r, b)) for r in range(P) for b in range(nb)]
    for t in th:
        t.start()
    for t in th:
        t.join(60)
    for t in timers:
        t.join(5)
    return errors


def test_protocol_random_delays():
    for seed, (P, nb) in enumerate([(2, 1), (3, 2), (4, 2), (8, 1)]):
        assert run_protocol(P, nb, R=10, ncols=5, seed=seed) == []


def test_protocol_slow_link():
    # rank 0's first push to rank 2 arrives long after everything else: rank 1
    # finishes reduction 1 and pushes reduction 2 to rank 2 in the meantime
    assert run_protocol(3, 1, R=6, ncols=3, seed=1, slow=(0, 2, 1, 0.3)) == []
    assert run_protocol(4, 2, R=6, ncols=4, seed=2, slow=(3, 0, 2, 0.3)) == []


def test_model_sees_the_single_counter_hazard():
    errs = run_protocol(3, 1, R=4, ncols=3, seed=1, per_parity=False, slow=(0, 2, 1, 0.3))
    assert errs and errs[0][0] == "stale" and errs[0][1] == 2
