"""BERT encoder layer whose GEMMs run on the uKernel executor (SURVEY §8 f-3:
"Epilogue fusion and a BERT-base PyTorch module swap").

The reference's dynamic-shape workload is a BERT encoder
at a varying sequence length: per layer four Dense operators (QKV, attention
output, FFN1 + bias + GELU, FFN2) and two BatchMatmuls (attention scores and
context). `EncoderLayer` keeps the torch module's parameters (bf16) and runs

  * every Dense through `Planner.dense` — the planner's uKernel plan for the
    current M = batch * seq, bias (and GELU for FFN1) fused into the epilogue;
  * both attention BatchMatmuls through `Planner.bmm` (batch = batch * heads);

softmax, layer norm and the residual adds stay in torch. `from_torch` copies
the weights of a `torch.nn.TransformerEncoderLayer`-like module with the
BERT layout (batch_first, post-norm, GELU). The attention scale 1/sqrt(d_head)
is folded into the Q rows of the QKV weight and bias (exact for d_head = 64:
a power of two), so the QKV epilogue already writes scaled queries; the
probability buffer's row padding is never read (the context BMM's K extent is
T: TMA zero-fills past it), so it is not cleared.
"""

from __future__ import annotations

import math

from .runtime import Planner


class EncoderLayer:
    def __init__(self, hidden: int = 768, heads: int = 12, ffn: int = 3072, planner: Planner | None = None,
                 device="cuda", seed: int = 0):
        import torch

        self.hidden, self.heads, self.ffn = hidden, heads, ffn
        self.planner = planner or Planner()
        g = torch.Generator(device="cpu").manual_seed(seed)

        def w(n, k):
            return (torch.randn(n, k, generator=g) / math.sqrt(k)).to(torch.bfloat16).to(device)

        def b(n):
            return (torch.randn(n, generator=g) * 0.02).to(torch.bfloat16).to(device)

        # nn.Linear layout [out, in] ("nk"): the weight is the K-major operand
        self.w_qkv, self.b_qkv = self._scale_q(w(3 * hidden, hidden), b(3 * hidden), hidden, heads)
        self.w_out, self.b_out = w(hidden, hidden), b(hidden)
        self.w_ffn1, self.b_ffn1 = w(ffn, hidden), b(ffn)
        self.w_ffn2, self.b_ffn2 = w(hidden, ffn), b(hidden)
        self.ln1 = (torch.ones(hidden, device=device, dtype=torch.bfloat16),
                    torch.zeros(hidden, device=device, dtype=torch.bfloat16))
        self.ln2 = (torch.ones(hidden, device=device, dtype=torch.bfloat16),
                    torch.zeros(hidden, device=device, dtype=torch.bfloat16))

    @staticmethod
    def _scale_q(w, b, hidden, heads):
        """Fold softmax's 1/sqrt(d_head) into the Q rows (the first `hidden`)."""
        scale = 1.0 / math.sqrt(hidden // heads)
        w, b = w.clone(), b.clone()
        w[:hidden] = (w[:hidden].float() * scale).to(w.dtype)
        b[:hidden] = (b[:hidden].float() * scale).to(b.dtype)
        return w, b

    @classmethod
    def from_torch(cls, layer, planner: Planner | None = None) -> "EncoderLayer":
        """Copy a torch.nn.TransformerEncoderLayer (batch_first, norm_first=False)."""
        import torch

        sa = layer.self_attn
        me = cls.__new__(cls)
        me.hidden = sa.embed_dim
        me.heads = sa.num_heads
        me.ffn = layer.linear1.out_features
        me.planner = planner or Planner()
        bf = lambda t: t.detach().to(torch.bfloat16).contiguous()  # noqa: E731
        me.w_qkv, me.b_qkv = cls._scale_q(bf(sa.in_proj_weight), bf(sa.in_proj_bias), me.hidden, me.heads)
        me.w_out, me.b_out = bf(sa.out_proj.weight), bf(sa.out_proj.bias)
        me.w_ffn1, me.b_ffn1 = bf(layer.linear1.weight), bf(layer.linear1.bias)
        me.w_ffn2, me.b_ffn2 = bf(layer.linear2.weight), bf(layer.linear2.bias)
        me.ln1 = (bf(layer.norm1.weight), bf(layer.norm1.bias))
        me.ln2 = (bf(layer.norm2.weight), bf(layer.norm2.bias))
        return me

    def __call__(self, x):
        """x: [batch, seq, hidden] bf16 -> same shape."""
        import torch
        import torch.nn.functional as F

        bsz, T, H = x.shape
        nh, hd = self.heads, H // self.heads
        pl = self.planner
        x2 = x.reshape(bsz * T, H).contiguous()
        qkv = pl.dense(x2, self.w_qkv, b_layout="nk", bias=self.b_qkv)              # [M, 3H]
        qkv = qkv.view(bsz, T, 3, nh, hd).permute(2, 0, 3, 1, 4)                    # [3, b, nh, T, hd]
        q = qkv[0].reshape(bsz * nh, T, hd).contiguous()                          # already scaled
        k = qkv[1].reshape(bsz * nh, T, hd).contiguous()
        v = qkv[2].reshape(bsz * nh, T, hd).contiguous()
        ldT = (T + 7) // 8 * 8                                                       # TMA 16-B row rule
        scores = torch.empty(bsz * nh, T, ldT, dtype=torch.bfloat16, device=x.device)
        pl.bmm(q, k, b_layout="nk", out=scores[:, :, :T])                           # Q K^T
        probs = torch.empty_like(scores)  # padding columns are never read
        probs[:, :, :T] = torch.softmax(scores[:, :, :T], dim=-1, dtype=torch.float32)
        ctx = pl.bmm(probs[:, :, :T], v, b_layout="kn", dynamic=("i", "k"))         # P V
        ctx = ctx.view(bsz, nh, T, hd).permute(0, 2, 1, 3).reshape(bsz * T, H).contiguous()
        attn = pl.dense(ctx, self.w_out, b_layout="nk", bias=self.b_out)
        h1 = F.layer_norm(x2 + attn, (H,), *self.ln1)                              # bf16 in, fp32 statistics
        f1 = pl.dense(h1, self.w_ffn1, b_layout="nk", bias=self.b_ffn1, activation="gelu")
        f2 = pl.dense(f1, self.w_ffn2, b_layout="nk", bias=self.b_ffn2)
        out = F.layer_norm(h1 + f2, (H,), *self.ln2)
        return out.view(bsz, T, H)
