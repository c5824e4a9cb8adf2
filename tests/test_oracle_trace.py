"""The oracle's optional DSI event trace (SPEC S:177-180 TraceEvent; SURVEY 8(c).2 "optional debug
outputs": a Fig. 1-style timeline), pinned against hand-derived schedules: DESIGN.md's worked
example (N 10, k 2, t_t 100, t_d 30, A = 110111101: segments 3, 5, 2, so rejections settle at
C(3) = 160 and 160 + C(5) = 380 and the last token at 540; with SP 1 the second task of a
segment waits for the first, giving 200, 500, 700) and Prop. 1's example (N 12, k 1,
t_d 14, t_t 100, A = 10111011111 -> 426)."""
import oracle as O


def pattern_index(bits: str) -> int:
    """Pattern mode: A_p = bit p-1 of the trial index (bits[0] is A_1)."""
    return sum(1 << i for i, b in enumerate(bits) if b == "1")


def kinds(ev, kind):
    return [e for e in ev if e["kind"] == kind]


def check_common(ev, N, sp, t_d):
    emitted = kinds(ev, "TokenEmitted")
    assert [e["position"] for e in emitted] == list(range(1, N + 1))  # every token once, in order
    assert all(a["time"] <= b["time"] for a, b in zip(emitted, emitted[1:]))
    # a documented total order, as SPEC S:178 asks (time, segment, kind)
    order = {k: i for i, k in enumerate(O.TRACE_KINDS)}
    keys = [(e["time"], e["segment"], order[e["kind"]]) for e in ev]
    assert keys == sorted(keys)
    # never more than SP target forwards in flight (Eq. 1's servers); a rejection
    # cancels the segment's threads, so the count is per segment
    busy, peak = {}, 0
    for e in ev:
        s = e["segment"]
        if e["kind"] == "VerifyDone":
            busy[s] -= 1
        elif e["kind"] == "VerifyDispatch":
            busy[s] = busy.get(s, 0) + 1
            peak = max(peak, busy[s])
    assert 1 <= peak <= sp
    # a draft is done before the target's verdict on it (Assumption 2, t_d <= t_t)
    done = {e["position"]: e["time"] for e in kinds(ev, "DraftDone")}
    for e in kinds(ev, "Accept") + kinds(ev, "Reject"):
        assert done[e["position"]] <= e["time"]
    return emitted


def test_worked_example_timeline_sp2():
    cfg = O.Config(100, 30, 0.5, 2, 2, 10, 0)
    rec, ev = O.trace(cfg, 0, pattern_index("110111101"), pattern=True)
    emitted = check_common(ev, 10, 2, 30)
    assert rec["dsi"] == 540 and emitted[-1]["time"] == 540
    assert [(e["time"], e["position"]) for e in kinds(ev, "Reject")] == [(160, 3), (380, 8)]
    assert [e["time"] for e in kinds(ev, "SegmentStart")] == [0, 160, 380]
    assert not kinds(ev, "VerifyQueued")  # Eq. 1 holds: 100 <= 2 * 2 * 30


def test_worked_example_timeline_sp1_queues():
    cfg = O.Config(100, 30, 0.5, 2, 1, 10, 0)
    rec, ev = O.trace(cfg, 0, pattern_index("110111101"), pattern=True)
    emitted = check_common(ev, 10, 1, 30)
    assert rec["dsi"] == 700 and emitted[-1]["time"] == 700
    assert [(e["time"], e["position"]) for e in kinds(ev, "Reject")] == [(200, 3), (500, 8)]
    # task 1 of the first segment is requested at 60 and waits for thread 0's server (FIFO, R7)
    q = kinds(ev, "VerifyQueued")
    assert q and q[0]["time"] == 60 and q[0]["thread"] == 1
    starts = [e for e in kinds(ev, "VerifyDispatch") if e["segment"] == 1]
    # thread 2 takes the server thread 1 releases at 200 -- the instant its rejection cancels it
    assert [(e["time"], e["thread"]) for e in starts] == [(0, 0), (100, 1), (200, 2)]


def test_proposition1_example_timeline():
    cfg = O.Config(100, 14, 0.5, 1, 8, 12, 0)
    rec, ev = O.trace(cfg, 0, pattern_index("10111011111"), pattern=True)
    emitted = check_common(ev, 12, 8, 14)
    assert rec["dsi"] == 426 and emitted[-1]["time"] == 426
    # rejections at positions 2 and 6 (A_2 = A_6 = 0), each costing one target forward
    assert [e["position"] for e in kinds(ev, "Reject")] == [2, 6]
    assert [e["time"] for e in kinds(ev, "Reject")] == [114, 256]  # C(2) = 100 + 14, then + C(4) = 100 + 3 * 14


def test_trace_matches_the_untraced_trial():
    cfg = O.Config(100, 7, 0.7, 3, 4, 60, 0)
    for i in range(20):
        rec, ev = O.trace(cfg, 2405141050, i)
        plain = O.trial(cfg, 2405141050, i)
        assert rec["dsi"] == plain["dsi"] and rec["si"] == plain["si"] and rec["m"] == plain["m"]
        assert len(kinds(ev, "Reject")) == plain["m"] - 1
        assert kinds(ev, "TokenEmitted")[-1]["time"] == plain["dsi"]
