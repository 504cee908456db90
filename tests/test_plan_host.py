"""Host-side work-plan logic of the split kernel (no GPU): attention.split_tail keeps every row
of every segment covered exactly once and renumbers the partial slots per unit in work-list
order, as dq_attention_plan does (csrc/attention.cu)."""

from paper_2405_12591_b200.attention import WorkPlan, split_tail


def _plan(items, seg_units, units):
    npt = [0] * units
    for s, _, _ in items:
        npt[seg_units[s]] += 1
    p0, acc = [], 0
    for u in range(units):
        p0.append(acc)
        acc += npt[u]
    cur, wpart = list(p0), []
    for s, _, _ in items:
        wpart.append(cur[seg_units[s]])
        cur[seg_units[s]] += 1
    return WorkPlan(len(items), acc, [x for it in items for x in it], wpart, p0, npt)


def test_split_tail_covers_rows_and_renumbers_slots():
    seg_units = [0, 1, 2, 0]                      # segment -> unit (unit 0 holds two segments)
    tiles = {0: 16, 1: 9, 2: 8, 3: 3}             # 64-row tiles per segment
    items = []
    for s, nt in tiles.items():
        t = 0
        while t < nt:
            n = min(8, nt - t)
            items.append((s, t * 64, n))
            t += n
    wp = _plan(items, seg_units, 3)
    out = split_tail(wp, seg_units, 3)
    assert out.nwork == wp.nwork + sum(1 for it in items[-3:] if it[2] >= 2)
    # rows covered exactly once per segment
    cover = {s: [] for s in tiles}
    for i in range(out.nwork):
        s, b0, t = out.work[3 * i: 3 * i + 3]
        cover[s] += list(range(b0 // 64, b0 // 64 + t))
    for s, nt in tiles.items():
        assert sorted(cover[s]) == list(range(nt))
    # the split items come last, whole items first in their original order
    assert out.work[: 3 * (wp.nwork - 3)] == wp.work[: 3 * (wp.nwork - 3)]
    # slots: unit u owns [p0, p0 + nparts), assigned in work-list order, each once
    assert out.total_parts == out.nwork == sum(out.unit_nparts)
    seen = {u: [] for u in range(3)}
    for i in range(out.nwork):
        seen[seg_units[out.work[3 * i]]].append(out.work_part[i])
    for u in range(3):
        assert seen[u] == list(range(out.unit_part0[u], out.unit_part0[u] + out.unit_nparts[u]))


def test_split_tail_zero_is_identity_and_single_tiles_stay_whole():
    seg_units = [0, 1]
    wp = _plan([(0, 0, 8), (1, 0, 1)], seg_units, 2)
    same = split_tail(wp, seg_units, 0)
    assert same.work == wp.work and same.work_part == wp.work_part
    one = split_tail(wp, seg_units, 1)            # the last item has one tile: nothing to split
    assert one.work == wp.work
