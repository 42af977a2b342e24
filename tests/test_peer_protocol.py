"""Model check of the peer transport's flag protocols (xdit_usp.cpp usp_call):
the ring K/V rotation and the Ulysses exchange.

The GPU tests run the real protocol with 2-8 processes; this CPU test explores it exhaustively-ish
under random interleavings of every rank's two streams, on a model that enqueues exactly the
operations usp_call enqueues for the ring (u = 1, r ranks, several consecutive calls):

  side stream, step s <= r-2:  wait credit[(s+1)&1] == 1; reset it; push my current block into
                               next's slot (s+1)&1; set next's data[(s+1)&1]; record ev_push[s]
  main stream, step s:         attention reads the current block (slot s&1, or the local block at
                               s = 0); if s <= r-2: wait ev_push[s]; post credit[s&1] to prev when
                               credit_after(s); wait data[(s+1)&1] == 1; reset it
                               (s = r-1: post credit[s&1] when credit_after(s))
  credit_after(s) = (s == 0 and r >= 3) or (1 <= s <= r-3) or s == last odd step;  credit[1] starts 1.

Checked: no deadlock; a push never overwrites a slot whose block the owner has not finished
reading; every read sees the block of the step it expects (ring index (i - s) mod r of this call);
flags end every call in their initial state.
"""
import random

import pytest


def credit_after(s, r):
    last_odd = r - 1 if (r - 1) % 2 else r - 2
    return (s == 0 and r >= 3) or (1 <= s <= r - 3) or s == last_odd


def build_program(i, r, calls):
    """Ops of rank i: two streams of (kind, args); 'event' ops give cross-stream ordering."""
    main, side = [], []
    for c in range(calls):
        # side stream starts after main reaches the step's start (ev_start), as in usp_call
        for s in range(r):
            main.append(("mark", (c, s)))  # ev_start of step s: the current block is in place
            if s <= r - 2:
                side.append(("wait_mark", (c, s)))
                side.append(("wait_flag", ("credit", (s + 1) & 1)))
                side.append(("reset", ("credit", (s + 1) & 1)))
                side.append(("push", (c, s)))
                side.append(("set_next", ("data", (s + 1) & 1)))
                side.append(("ev_push", (c, s)))
            main.append(("read", (c, s)))
            if s <= r - 2:
                main.append(("wait_ev_push", (c, s)))
                if credit_after(s, r):
                    main.append(("set_prev", ("credit", s & 1)))
                main.append(("wait_flag", ("data", (s + 1) & 1)))
                main.append(("reset", ("data", (s + 1) & 1)))
            elif credit_after(s, r):
                main.append(("set_prev", ("credit", s & 1)))
    return main, side


def simulate(r, calls, seed):
    rng = random.Random(seed)
    flags = [{("data", 0): 0, ("data", 1): 0, ("credit", 0): 0, ("credit", 1): 1} for _ in range(r)]
    # slot contents: (call, ring index of the block); "local" block is separate
    slot = [[None, None] for _ in range(r)]
    marks = [set() for _ in range(r)]
    evs = [set() for _ in range(r)]
    progs = [build_program(i, r, calls) for i in range(r)]
    pc = [[0, 0] for _ in range(r)]
    pending_read = [[[] for _ in range(2)] for _ in range(r)]  # blocks the owner still has to read

    def cur_block(i, c, s):
        return (c, (i - s) % r)

    def try_step(i, st):
        prog = progs[i][st]
        if pc[i][st] >= len(prog):
            return False
        kind, arg = prog[pc[i][st]]
        nxt, prv = (i + 1) % r, (i - 1) % r
        if kind == "mark":
            marks[i].add(arg)
        elif kind == "wait_mark":
            if arg not in marks[i]:
                return False
        elif kind == "wait_flag":
            if flags[i][arg] < 1:
                return False
        elif kind == "reset":
            flags[i][arg] = 0
        elif kind == "push":
            c, s = arg
            b = (s + 1) & 1
            # safety: next must have read whatever it was supposed to read from slot b
            assert not pending_read[nxt][b], f"rank {i} overwrote slot {b} of {nxt} before it was read"
            block = cur_block(i, c, s)  # my current block (local at s = 0, else slot s&1)
            if s >= 1:
                assert slot[i][s & 1] == block, "pushed a block other than the current one"
            slot[nxt][b] = block
            pending_read[nxt][b].append((c, s + 1))
        elif kind == "set_next":
            assert flags[nxt][arg] == 0, f"lost signal: {arg} on {nxt} already set"
            flags[nxt][arg] = 1
        elif kind == "set_prev":
            assert flags[prv][arg] == 0, f"lost credit: {arg} on {prv} already set"
            flags[prv][arg] = 1
        elif kind == "ev_push":
            evs[i].add(arg)
        elif kind == "wait_ev_push":
            if arg not in evs[i]:
                return False
        elif kind == "read":
            c, s = arg
            if s >= 1:
                b = s & 1
                assert pending_read[i][b] and pending_read[i][b][0] == (c, s), "read without matching data"
                assert slot[i][b] == cur_block(i, c, s), "read the wrong block"
                pending_read[i][b].pop(0)
        pc[i][st] += 1
        return True

    while True:
        moves = [(i, st) for i in range(r) for st in (0, 1)]
        rng.shuffle(moves)
        if not any(try_step(i, st) for i, st in moves):
            break
    done = all(pc[i][st] == len(progs[i][st]) for i in range(r) for st in (0, 1))
    assert done, f"deadlock: pcs {pc}"
    for i in range(r):  # flags back in their initial state
        assert flags[i] == {("data", 0): 0, ("data", 1): 0, ("credit", 0): 0, ("credit", 1): 1}, flags[i]


@pytest.mark.parametrize("r", [2, 3, 4, 5, 8])
def test_ring_flag_protocol(r):
    for seed in range(200):
        simulate(r, calls=3, seed=seed)


def test_credit_posts_match_pushes():
    """Per call, a rank posts exactly as many credits per slot as its predecessor pushes into it."""
    for r in range(2, 9):
        posts = [0, 0]
        for s in range(r):
            if credit_after(s, r):
                posts[s & 1] += 1
        pushes = [0, 0]
        for s in range(r - 1):
            pushes[(s + 1) & 1] += 1
        assert posts == pushes, (r, posts, pushes)


def simulate_ulysses(u, calls, seed):
    """Model of the Ulysses exchange (one stream per rank): pack = stores into every peer's receive
    chunk [me], set A2A[me] on each peer, wait + reset my A2A[p] for all p != me, unpack (reads my
    receive buffer), epilogue = stores into every peer's O chunk [me], set O[me] on each peer, wait +
    reset my O[p], unpack_out (reads my O buffer)."""
    rng = random.Random(seed)
    flags = [{(k, p): 0 for k in ("a2a", "o") for p in range(u)} for _ in range(u)]
    recv = [[None] * u for _ in range(u)]   # recv[owner][writer] = call of the chunk
    orecv = [[None] * u for _ in range(u)]
    unread = [[False] * u for _ in range(u)]
    ounread = [[False] * u for _ in range(u)]
    prog = []
    for i in range(u):
        ops = []
        for c in range(calls):
            ops.append(("pack", c))
            ops += [("set", ("a2a", p)) for p in range(u) if p != i]
            for p in range(u):
                if p != i:
                    ops += [("wait", ("a2a", p)), ("reset", ("a2a", p))]
            ops.append(("unpack", c))
            ops.append(("epilogue", c))
            ops += [("set", ("o", p)) for p in range(u) if p != i]
            for p in range(u):
                if p != i:
                    ops += [("wait", ("o", p)), ("reset", ("o", p))]
            ops.append(("unpack_out", c))
        prog.append(ops)
    pc = [0] * u

    def step(i):
        if pc[i] >= len(prog[i]):
            return False
        kind, a = prog[i][pc[i]]
        if kind == "pack":
            for p in range(u):
                assert not unread[p][i], f"rank {i} overwrote {p}'s receive chunk before it was unpacked"
                recv[p][i], unread[p][i] = a, True
        elif kind == "set":
            k, p = a
            assert flags[p][(k, i)] == 0, "lost signal"
            flags[p][(k, i)] = 1
        elif kind == "wait":
            if flags[i][a] < 1:
                return False
        elif kind == "reset":
            flags[i][a] = 0
        elif kind == "unpack":
            assert all(recv[i][p] == a for p in range(u)), "unpacked a chunk of another call"
            unread[i] = [False] * u
        elif kind == "epilogue":
            for p in range(u):
                assert not ounread[p][i], f"rank {i} overwrote {p}'s O chunk before it was unpacked"
                orecv[p][i], ounread[p][i] = a, True
        elif kind == "unpack_out":
            assert all(orecv[i][p] == a for p in range(u)), "unpacked an O chunk of another call"
            ounread[i] = [False] * u
        pc[i] += 1
        return True

    while True:
        order = list(range(u))
        rng.shuffle(order)
        if not any(step(i) for i in order):
            break
    assert pc == [len(p) for p in prog], f"deadlock: {pc}"
    assert all(v == 0 for f in flags for v in f.values())


@pytest.mark.parametrize("u", [2, 3, 4, 8])
def test_ulysses_flag_protocol(u):
    for seed in range(200):
        simulate_ulysses(u, calls=3, seed=seed)
