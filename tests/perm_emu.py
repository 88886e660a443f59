"""CPU emulation of k_perm's word-gather tables (TEST INFRASTRUCTURE ONLY).

Reads a span plan through ``mpx_plan_dump`` and replays, byte for byte, what
the kernel does with it (csrc/k_perm.cu ``permute``): the chunk's input
staged at its 16-byte phase in a buffer with front slack, each table slot's
4 input bytes fetched through its window selectors (word form) or byte
deltas (byte form), and the store rules for whole, edge and gap words.  The
tests compare the result with the oracle, so the host lowering (tables,
phases, periods) is checked without a GPU.
"""

import ctypes

import numpy as np

K_FRONT = 16
K_STAGE = 3072                             # desc.cuh kSpanStage: bytes staged per chunk


def dump(mp, dt, count=1):
    lib = mp._lib.lib
    n = ctypes.c_int64()
    lib.mpx_plan_dump(dt._h, count, None, 0, ctypes.byref(n))
    buf = (ctypes.c_int64 * n.value)()
    mp._lib.check(lib.mpx_plan_dump(dt._h, count, buf, n.value, ctypes.byref(n)))
    v = list(buf)
    pos = 0

    def take(k):
        nonlocal pos
        out = v[pos:pos + k]
        pos += k
        return out

    kind, depth = take(2)
    outer = [tuple(take(3)) for _ in range(2)][:depth]
    (nch,) = take(1)
    chunks = [dict(zip(("src", "pk", "span", "plen", "n", "body", "stride", "uperm", "pperm"), take(9)))
              for _ in range(nch)]
    (nspec,) = take(1)
    specs = []
    for _ in range(nspec):
        W, Dw, ns, mode, tab = take(5)
        specs.append({"W": W, "Dw": Dw, "ns": ns, "bytes": mode == 1, "tab": tab, "wc": take(16)})
    (ntab,) = take(1)
    tab = [tuple(take(4)) for _ in range(ntab)]
    return {"kind": kind, "outer": outer, "chunks": chunks, "specs": specs, "tab": tab}


def _s16(x):
    x &= 0xFFFF
    return x - 0x10000 if x & 0x8000 else x


def _units(plan):
    """(layout offset, packed offset) of every (outer index, chunk) unit."""
    offs = [(0, 0)]
    for cnt, st, pk in reversed(plan["outer"]):   # innermost outer level varies fastest
        offs = [(o * st + lo, o * pk + po) for o in range(cnt) for lo, po in offs]
    offs.sort(key=lambda t: t[1])
    return offs


def run(plan, pack, src, dst, src_addr=0, dst_addr=0, limit=None):
    """Apply the plan like k_perm: pack (layout src -> packed dst) or unpack.
    src/dst are uint8 arrays; *_addr are the buffers' device addresses mod 16."""
    total = sum(c["plen"] for c in plan["chunks"]) * max(1, len(_units(plan)))
    limit = total if limit is None else limit
    for loff, poff in _units(plan):
        for c in plan["chunks"]:
            lay0, pk0 = c["src"] + loff, c["pk"] + poff
            if pk0 >= limit:
                continue
            spec = plan["specs"][c["pperm"] if pack else c["uperm"]]
            avail = min(c["plen"], limit - pk0)
            if pack:
                in_off, in_len, out_off, out_len, full = lay0, c["span"], pk0, avail, True
                in_addr, out_addr = src_addr + lay0, dst_addr + pk0
            else:
                in_off, in_len, out_off, out_len, full = pk0, avail, lay0, c["span"], avail >= c["plen"]
                in_addr, out_addr = src_addr + pk0, dst_addr + lay0
            _chunk(spec, plan["tab"], src, in_off, in_len, in_addr, dst, out_off, out_len, out_addr, full)


def _chunk(spec, tab, src, in_off, in_len, in_addr, dst, out_off, out_len, out_addr, full):
    a = in_addr & 15
    ap, po = a & 3, out_addr & 3
    # staged buffer: front slack, then the 16-byte blocks holding the input
    buf = np.full(K_FRONT + K_STAGE + 32 + 64, 0xEE, np.uint8)
    lo = in_off - a
    nv = (a + in_len + 15) >> 4
    for k in range(16 * nv):
        if 0 <= lo + k < src.size:
            buf[K_FRONT + k] = src[lo + k]
    A = K_FRONT + (a & ~3)                 # index of input word 0
    W, Dw4 = spec["W"], 4 * spec["Dw"]
    wc = spec["wc"][po * 4 + ap]
    ents = tab[spec["tab"] + (po * 4 + ap) * W: spec["tab"] + (po * 4 + ap) * W + wc]
    words = (po + out_len + 3) >> 2
    kw, kd = 0, 0
    while kw < words:
        for x, lo_w, hi_w, mix in ents:
            x = x - (1 << 32) if x >= (1 << 31) else x      # int32 window / byte-0 offset
            j, cov = lo_w >> 24, (lo_w >> 16) & 0xF
            gw = kw + j
            if gw >= words:
                continue
            base = A + x + kd
            vals, offs = [], []
            for i in range(4):
                if spec["bytes"]:
                    d = [0, _s16(hi_w), _s16(hi_w >> 16), _s16(mix)][i]
                    p = base + d
                else:
                    pr = (lo_w >> (20 + i)) & 1
                    sel = (hi_w if pr else lo_w)
                    nib = (sel >> (4 * i)) & 7
                    p = base + 8 * pr + 4 * (nib >> 2) + (nib & 3)
                offs.append(p - A - ap)              # input byte offset
                vals.append(buf[p] if 0 <= p < buf.size else 0xEE)
            for i in range(4):
                if not (cov >> i) & 1:
                    continue
                q = 4 * gw + i - po
                if q < 0 or q >= out_len:
                    continue
                if not full and offs[i] >= in_len:
                    continue
                dst[out_off + q] = vals[i]
        kw += W
        kd += Dw4
