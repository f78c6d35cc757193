"""Emit csrc/median_block.cuh: one min/max network that computes the exact 5x5
medians of a TW x TH block of adjacent outputs, sharing work between them.

Construction (selection by rank bounds on sorted shared sets):
  * every sorted set is a rectangle of input cells, built by Batcher odd-even
    merges of memoised halves split at power-of-two-aligned rows/columns, so
    neighbouring outputs reuse the same sorted column pieces;
  * the output block is split recursively (longer side first); at each node
    the cells common to every window of the node are merged into a sorted list
    L, and L is trimmed to the ranks that can still be a window median: with
    dlo cells known <= and dhi known >= the median and r = 25 - dlo - dhi - |L|
    cells not yet seen, only L[12 - dlo - r .. 12 - dlo] can be it;
  * at a single output the unseen cells E are sorted and the median is the
    k-th element of L u E: min_i max(L[k - i], E[i - 1]).
Dead min/max outputs are pruned backwards from the median wires.  The network
is checked here against sorted windows on random real and tied inputs (min/max
networks obey the 0-1 principle; tests/test_gpu_ops.py and the pipeline tests
check the CUDA result bit for bit against the oracle).
"""
from __future__ import annotations

import random
import sys
from pathlib import Path

sys.setrecursionlimit(100000)
K, MID = 5, 12


class Net:
    def __init__(self):
        self.ops, self.nw = [], 0

    def new(self):
        self.nw += 1
        return self.nw - 1

    def mx(self, a, b):
        o = self.new()
        self.ops.append(("max", a, b, o))
        return o

    def mn(self, a, b):
        o = self.new()
        self.ops.append(("min", a, b, o))
        return o

    def cs(self, a, b):
        return self.mn(a, b), self.mx(a, b)


def omerge(net, A, B):
    """Batcher odd-even merge of sorted A and B, any sizes."""
    if not A:
        return list(B)
    if not B:
        return list(A)
    if len(A) == 1 and len(B) == 1:
        return list(net.cs(A[0], B[0]))
    E = omerge(net, A[0::2], B[0::2])
    O = omerge(net, A[1::2], B[1::2])
    res, i = [E[0]], 0
    while i < len(O) or i + 1 < len(E):
        if i < len(O) and i + 1 < len(E):
            res += list(net.cs(O[i], E[i + 1]))
        elif i < len(O):
            res.append(O[i])
        else:
            res.append(E[i + 1])
        i += 1
    return res


def split_point(a, b):
    for p in range(10, -1, -1):
        s = 1 << p
        m = ((a // s) + 1) * s
        if a < m <= b:
            return m
    return (a + b + 1) // 2


def build(TW, TH):
    net = Net()
    inp = {(x, y): net.new() for y in range(TH + K - 1) for x in range(TW + K - 1)}
    memo = {}

    def srect(x0, x1, y0, y1):  # sorted cells of the inclusive rectangle
        key = (x0, x1, y0, y1)
        if key not in memo:
            if x0 == x1 and y0 == y1:
                r = [inp[(x0, y0)]]
            elif x0 == x1:
                m = split_point(y0, y1)
                r = omerge(net, srect(x0, x1, y0, m - 1), srect(x0, x1, m, y1))
            else:
                m = split_point(x0, x1)
                r = omerge(net, srect(x0, m - 1, y0, y1), srect(m, x1, y0, y1))
            memo[key] = r
        return memo[key]

    def common(block):
        xs = [b[0] for b in block]
        ys = [b[1] for b in block]
        c = (max(xs), min(xs) + K - 1, max(ys), min(ys) + K - 1)
        return c if c[0] <= c[1] and c[2] <= c[3] else None

    def minus(big, small):  # big \ small as rectangles (small shares big's span on one axis)
        if small is None:
            return [big]
        x0, x1, y0, y1 = big
        a0, a1, b0, b1 = small
        res = []
        if a0 > x0:
            res.append((x0, a0 - 1, y0, y1))
        if a1 < x1:
            res.append((a1 + 1, x1, y0, y1))
        if b0 > y0:
            res.append((max(x0, a0), min(x1, a1), y0, b0 - 1))
        if b1 < y1:
            res.append((max(x0, a0), min(x1, a1), b1 + 1, y1))
        return [r for r in res if r[0] <= r[1] and r[2] <= r[3]]

    outs = {}

    def solve(block, L, dlo, dhi, done):
        r = K * K - dlo - dhi - len(L)
        lo, hi = max(0, MID - dlo - r), min(len(L) - 1, MID - dlo)
        dhi += len(L) - 1 - hi
        dlo += lo
        L = L[lo:hi + 1]
        if len(block) == 1:
            (xo, yo), = block
            E = []
            for rc in minus((xo, xo + K - 1, yo, yo + K - 1), done):
                E = omerge(net, E, srect(*rc)) if E else srect(*rc)
            k, best = MID - dlo, None
            for i in range(max(0, k + 1 - len(L)), min(len(E), k + 1) + 1):
                parts = ([L[k - i]] if k - i >= 0 else []) + ([E[i - 1]] if i >= 1 else [])
                v = parts[0] if len(parts) == 1 else net.mx(parts[0], parts[1])
                best = v if best is None else net.mn(best, v)
            outs[(xo, yo)] = best
            return
        xs = sorted({b[0] for b in block})
        ys = sorted({b[1] for b in block})
        if len(xs) >= len(ys):
            h = len(xs) // 2
            parts = [[b for b in block if b[0] in xs[:h]], [b for b in block if b[0] in xs[h:]]]
        else:
            h = len(ys) // 2
            parts = [[b for b in block if b[1] in ys[:h]], [b for b in block if b[1] in ys[h:]]]
        for sub in parts:
            c = common(sub)
            L2 = L
            if c is not None:
                for rc in minus(c, done):
                    L2 = omerge(net, L2, srect(*rc))
            solve(sub, L2, dlo, dhi, c if c is not None else done)

    block = [(x, y) for y in range(TH) for x in range(TW)]
    c = common(block)
    solve(block, srect(*c) if c else [], 0, 0, c)
    out_list = [outs[b] for b in block]
    need, kept = set(out_list), []
    for op in reversed(net.ops):
        if op[3] in need:
            kept.append(op)
            need.update((op[1], op[2]))
    return inp, out_list, kept[::-1], block


def check(inp, outs, kept, block, trials=400, seed=1):
    rnd = random.Random(seed)
    for t in range(trials):
        v = {w: (float(rnd.randrange(1 + t % 4)) if t % 3 else rnd.random()) for w in inp.values()}
        for op, a, b, o in kept:
            v[o] = max(v[a], v[b]) if op == "max" else min(v[a], v[b])
        for (xo, yo), o in zip(block, outs):
            win = sorted(v[inp[(x, y)]] for y in range(yo, yo + K) for x in range(xo, xo + K))
            assert v[o] == win[MID], (t, xo, yo)


def emit(TW, TH):
    inp, outs, kept, block = build(TW, TH)
    check(inp, outs, kept, block)
    used = {w for op in kept for w in op[1:3]} | set(outs)
    name = {w: f"i{y}_{x}" for (x, y), w in inp.items()}
    body = [f"  const float {name[w]} = t[{y} * stride + {x}];"
            for (x, y), w in sorted(inp.items(), key=lambda kv: (kv[0][1], kv[0][0])) if w in used]
    for k, (op, a, b, o) in enumerate(kept):
        name[o] = f"m{k}"
        body.append(f"  const float m{k} = {'fmaxf' if op == 'max' else 'fminf'}({name[a]}, {name[b]});")
    body += [f"  out[{yo}][{xo}] = {name[o]};" for (xo, yo), o in zip(block, outs)]
    return len(kept), body


def main():
    TW, TH = (int(v) for v in sys.argv[1:3]) if len(sys.argv) >= 3 else (8, 2)
    n, body = emit(TW, TH)
    text = [
        "// GENERATED by tools/gen_median_blocks.py -- do not edit.",
        f"// Exact 5x5 medians of a {TW}x{TH} block of adjacent outputs with one shared",
        f"// min/max network: {n} ops ({n / (TW * TH):.1f} per output; a separate pruned",
        "// median-of-25 network per output needs ~200).",
        "#pragma once",
        "",
        f"constexpr int kMedBlockW = {TW}, kMedBlockH = {TH};",
        "",
        "// t: top-left input cell of the block's (TW+4) x (TH+4) window, row stride `stride`",
        "__device__ __forceinline__ void median5_block(const float* __restrict__ t, int stride,",
        f"                                              float (&out)[{TH}][{TW}]) {{",
        *body,
        "}",
        "",
    ]
    Path(__file__).resolve().parent.parent.joinpath("csrc", "median_block.cuh").write_text("\n".join(text))
    print(f"{TW}x{TH}: {n} ops")


if __name__ == "__main__":
    main()
