"""Authored model graphs for the paper's benchmarks.

The reference ships only miniature generators; the paper's graphs (NasRNN,
BERT, ResNeXt-50, SqueezeNet, NasNet-A, Inception-v3) are
written here in the 20-operator language of tensor_lang.py, following the
structure of the TASO benchmark definitions the paper used.  Operators the
language lacks (softmax, layer-norm, batch-norm) are omitted exactly as in
TASO's own BERT/NasRNN examples; shapes are chosen so every node
shape-checks.  Graphs are deterministic (no randomness).
"""

from __future__ import annotations

from .tensor_lang import TensorGraph, make_identifier as ident, make_single_rooted


class _B:
    """Small builder with auto-numbered node names."""

    def __init__(self):
        self.g = TensorGraph()
        self.k = 0

    def name(self, tag: str) -> str:
        self.k += 1
        return f"{tag}{self.k}"

    def input(self, shape, tag="x"):
        n = self.name(tag)
        return self.g.add(n, "input", identifier=ident(n, shape))

    def weight(self, shape, tag="w"):
        n = self.name(tag)
        return self.g.add(n, "weight", identifier=ident(n, shape))

    def op(self, op, inputs, tag=None, **params):
        return self.g.add(self.name(tag or op), op, tuple(inputs), **params)

    def matmul(self, a, b, act=0):
        return self.op("matmul", (a, b), activation=act)

    def conv(self, x, w, stride=1, pad=0, act=0):
        return self.op("conv", (x, w), stride_h=stride, stride_w=stride, padding=pad, activation=act)

    def pool(self, kind, x, k, stride, pad=0):
        return self.op(kind, (x,), kernel_h=k, kernel_w=k, stride_h=stride, stride_w=stride,
                       padding=pad, activation=0)

    def done(self, outputs):
        self.g.set_outputs(list(outputs))
        return make_single_rooted(self.g)


def bert(layers: int = 12, seq: int = 64, hidden: int = 768, heads: int = 12, ffn: int = 3072) -> TensorGraph:
    """BERT-base encoder stack (TASO examples/bert.py structure: shared-input
    Q/K/V projections, per-head reshape/transpose, batched attention matmuls,
    output projection, residual adds; plus the FFN with relu)."""
    b = _B()
    dh = hidden // heads
    x = b.input((seq, hidden), "x")
    x = b.op("relu", (x,))
    for _ in range(layers):
        q = b.matmul(x, b.weight((hidden, hidden), "wq"))
        k = b.matmul(x, b.weight((hidden, hidden), "wk"))
        v = b.matmul(x, b.weight((hidden, hidden), "wv"))
        q = b.op("reshape", (q,), shape=f"{seq}_{heads}_{dh}")
        k = b.op("reshape", (k,), shape=f"{seq}_{heads}_{dh}")
        v = b.op("reshape", (v,), shape=f"{seq}_{heads}_{dh}")
        q = b.op("transpose", (q,), perm="1_0_2")
        k = b.op("transpose", (k,), perm="1_2_0")
        v = b.op("transpose", (v,), perm="1_0_2")
        logits = b.matmul(q, k)
        ctx = b.matmul(logits, v)
        ctx = b.op("transpose", (ctx,), perm="1_0_2")
        ctx = b.op("reshape", (ctx,), shape=f"{seq}_{hidden}")
        att = b.matmul(ctx, b.weight((hidden, hidden), "wo"))
        r1 = b.op("ewadd", (x, att))
        h = b.op("relu", (b.matmul(r1, b.weight((hidden, ffn), "w1")),))
        f = b.matmul(h, b.weight((ffn, hidden), "w2"))
        x = b.op("ewadd", (r1, f))
    return b.done([x])


def nasrnn(steps: int = 5, batch: int = 1, hidden: int = 512) -> TensorGraph:
    """NASNet RNN cell unrolled (TASO examples/nasrnn.py structure): eight
    input and eight hidden projections per step sharing x_t / h_t, combined by
    ewadd / ewmul / sigmoid / tanh / relu."""
    b = _B()
    h = b.input((batch, hidden), "h")
    for _ in range(steps):
        x = b.input((batch, hidden), "xt")
        mx = [b.matmul(x, b.weight((hidden, hidden), "wx")) for _ in range(8)]
        mh = [b.matmul(h, b.weight((hidden, hidden), "wh")) for _ in range(8)]
        s = [b.op("ewadd", (mx[i], mh[i])) for i in range(8)]
        a = [b.op("sigmoid", (s[0],)), b.op("relu", (s[1],)), b.op("sigmoid", (s[2],)), b.op("relu", (s[3],)),
             b.op("tanh", (s[4],)), b.op("sigmoid", (s[5],)), b.op("tanh", (s[6],)), b.op("relu", (s[7],))]
        m = [b.op("ewmul", (a[0], a[1])), b.op("ewadd", (a[2], a[3])), b.op("ewmul", (a[4], a[5])),
             b.op("ewadd", (a[6], a[7]))]
        n1 = b.op("tanh", (b.op("ewmul", (m[0], m[1])),))
        n2 = b.op("tanh", (b.op("ewadd", (m[2], m[3])),))
        h = b.op("ewmul", (n1, n2))
    return b.done([h])


def squeezenet(hw: int = 56, fires=((96, 16, 64), (128, 16, 64), (128, 32, 128), (256, 32, 128),
                                   (256, 48, 192), (384, 48, 192), (384, 64, 256), (512, 64, 256))) -> TensorGraph:
    """SqueezeNet 1.0 fire modules: 1x1 squeeze, then 1x1 and 3x3 expands on the
    same input concatenated on channels (conv-merge-* candidates)."""
    b = _B()
    x = b.input((1, 3, hw * 4, hw * 4), "img")
    x = b.conv(x, b.weight((96, 3, 7, 7)), stride=2, pad=0, act=1)
    x = b.pool("poolmax", x, 3, 2)
    c = 96
    for i, (cin, sq, ex) in enumerate(fires):
        s = b.conv(x, b.weight((sq, c, 1, 1)), act=1)
        e1 = b.conv(s, b.weight((ex, sq, 1, 1)), act=1)
        e3 = b.conv(s, b.weight((ex, sq, 3, 3)), act=1)
        x = b.op("concat_2", (e1, e3), axis=1)
        c = 2 * ex
        if i in (2, 6):
            x = b.pool("poolmax", x, 3, 2)
    x = b.conv(x, b.weight((1000, c, 1, 1)), act=1)
    x = b.pool("poolavg", x, 13, 1, pad=0)
    return b.done([x])


def resnext50(hw: int = 56, blocks=(3, 4, 6, 3), groups: int = 32) -> TensorGraph:
    """ResNeXt-50 (32x4d): bottleneck blocks with grouped 3x3 convs, relu and
    residual ewadd; projection shortcuts on the first block of each stage."""
    b = _B()
    x = b.input((1, 64, hw, hw), "img")
    c = 64
    width = 128
    out = 256
    for si, nb in enumerate(blocks):
        for bi in range(nb):
            stride = 2 if (bi == 0 and si > 0) else 1
            t = b.conv(x, b.weight((width, c, 1, 1)), act=1)
            t = b.conv(t, b.weight((width, width // groups, 3, 3)), stride=stride, act=1)
            t = b.conv(t, b.weight((out, width, 1, 1)))
            if bi == 0:
                sc = b.conv(x, b.weight((out, c, 1, 1)), stride=stride)
            else:
                sc = x
            x = b.op("relu", (b.op("ewadd", (t, sc)),))
            c = out
        width *= 2
        out *= 2
    return b.done([x])


def inception_v3(hw: int = 35, blocks: int = 3) -> TensorGraph:
    """Inception-v3 style A/B/C modules: parallel 1x1, 1x1->3x3, 1x1->3x3->3x3
    and pool->1x1 branches over a shared input, concatenated on channels."""
    b = _B()
    x = b.input((1, 192, hw, hw), "img")
    c = 192
    for i in range(blocks):
        b1 = b.conv(x, b.weight((64, c, 1, 1)), act=1)
        b3 = b.conv(x, b.weight((48, c, 1, 1)), act=1)
        b3 = b.conv(b3, b.weight((64, 48, 5, 5)), act=1)
        b5 = b.conv(x, b.weight((64, c, 1, 1)), act=1)
        b5 = b.conv(b5, b.weight((96, 64, 3, 3)), act=1)
        b5 = b.conv(b5, b.weight((96, 96, 3, 3)), act=1)
        bp = b.pool("poolavg", x, 3, 1)
        bp = b.conv(bp, b.weight((32 if i == 0 else 64, c, 1, 1)), act=1)
        x = b.op("concat_4", (b1, b3, b5, bp), axis=1)
        c = 64 + 64 + 96 + (32 if i == 0 else 64)
    # reduction + C-style modules with 1x1 branches sharing the input
    for _ in range(2):
        r1 = b.conv(x, b.weight((192, c, 1, 1)), act=1)
        r2 = b.conv(x, b.weight((192, c, 1, 1)), act=1)
        r2 = b.conv(r2, b.weight((192, 192, 3, 3)), act=1)
        r3 = b.conv(x, b.weight((192, c, 1, 1)), act=1)
        rp = b.conv(b.pool("poolmax", x, 3, 1), b.weight((192, c, 1, 1)), act=1)
        x = b.op("concat_4", (r1, r2, r3, rp), axis=1)
        c = 768
    return b.done([x])


def nasnet_a(hw: int = 32, cells: int = 4, c: int = 64) -> TensorGraph:
    """NasNet-A normal cells: several branches of (separable-style) convs and
    pools over two shared inputs, combined pairwise with ewadd and
    concatenated (many shared-input conv merges)."""
    b = _B()
    prev = b.input((1, c, hw, hw), "img")
    cur = b.conv(prev, b.weight((c, c, 1, 1)), act=1)
    for _ in range(cells):
        h0 = b.conv(prev, b.weight((c, c, 1, 1)), act=1)
        h1 = b.conv(cur, b.weight((c, c, 1, 1)), act=1)
        y1 = b.op("ewadd", (b.conv(h1, b.weight((c, c, 3, 3))), b.conv(h1, b.weight((c, c, 5, 5)))))
        y2 = b.op("ewadd", (b.conv(h0, b.weight((c, c, 3, 3))), b.conv(h1, b.weight((c, c, 3, 3)))))
        y3 = b.op("ewadd", (b.pool("poolavg", h1, 3, 1), h0))
        y4 = b.op("ewadd", (b.pool("poolavg", h0, 3, 1), b.pool("poolavg", h0, 3, 1)))
        y5 = b.op("ewadd", (b.conv(h0, b.weight((c, c, 5, 5))), b.conv(h0, b.weight((c, c, 3, 3)))))
        out = b.op("concat_6", (h1, y1, y2, y3, y4, y5), axis=1)
        prev, cur = cur, b.conv(out, b.weight((c, 6 * c, 1, 1)), act=1)
    return b.done([cur])


MODELS = {
    "nasrnn": nasrnn,
    "bert": bert,
    "resnext50": resnext50,
    "squeezenet": squeezenet,
    "nasnet_a": nasnet_a,
    "inception_v3": inception_v3,
}
