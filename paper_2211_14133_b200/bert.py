"""BERT encoder stages for the PipeFisher runtime (the F/B work that creates
the pipeline bubbles; SURVEY.md §2.4 last row).

F/B is plain PyTorch (cuBLAS bf16 GEMMs, SDPA attention) — it is not a
hot-path kernel of this repo.  What matters for the K-FAC path is the tape
capture: every K-FAC linear (Q, K, V, O, FFN1, FFN2 of each encoder layer)
records its input ``a`` and output gradient ``e`` for the micro-batches of
the refresh cycle's first step (reference BatchTape, kfac.hpp:33-37; SURVEY
A.5), as bf16 ``[n_tokens x d]`` exactly as the forward / backward produce
it — the SYRK reads it in place as an MN-major operand (no transpose).  Q/K/V share one
input, so the A-set of a layer has 4 distinct tapes for 6 factors.

A stage owns a contiguous run of encoder layers, plus the embeddings (first
stage) or the masked-LM head (last stage).  Weights are fp32 masters; the
forward runs under bf16 autocast.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import torch
import torch.nn.functional as F
from torch import nn

# (name, input tape key, d_in, d_out) of the K-FAC linears of one layer
LINEARS = ("q", "k", "v", "o", "ffn1", "ffn2")


@dataclass
class BertConfig:
    hidden: int = 1024
    ffn: int = 4096
    heads: int = 16
    layers: int = 24
    vocab: int = 30522
    max_pos: int = 512
    mlm_fraction: float = 0.15

    @staticmethod
    def large() -> "BertConfig":
        return BertConfig()

    @staticmethod
    def base() -> "BertConfig":
        return BertConfig(hidden=768, ffn=3072, heads=12, layers=12)


class TapeStore:
    """Per-stage tape buffers of one refresh cycle: tapes[(layer, key, micro)]
    -> bf16 [d x n].  key: 'a_qkv','a_o','a_ffn1','a_ffn2' (A-set) and
    'e_q','e_k','e_v','e_o','e_ffn1','e_ffn2' (B-set)."""

    def __init__(self):
        self.tapes: Dict[Tuple[int, str, int], torch.Tensor] = {}
        self.active_micro: Optional[int] = None

    def put(self, layer: int, key: str, x2d: torch.Tensor):
        if self.active_micro is None:
            return
        # token-major [n x d] as produced (features contiguous): the SYRK reads
        # it in place as an MN-major tensor-core operand -- no transposed copy
        # (a view of the bf16 activation when it already is one)
        x2d = x2d.detach()
        if x2d.dtype != torch.bfloat16:
            x2d = x2d.to(torch.bfloat16)
        if x2d.stride(1) != 1 or x2d.stride(0) % 8 != 0 or x2d.data_ptr() % 16 != 0:
            x2d = x2d.contiguous()
        self.tapes[(layer, key, self.active_micro)] = x2d

    def get(self, layer: int, key: str, micro: int) -> torch.Tensor:
        return self.tapes[(layer, key, micro)]

    def clear(self):
        self.tapes.clear()


class _TapedLinear(torch.autograd.Function):
    """y = x W^T + b, recording a = x (forward) and e = dL/dy (backward)."""

    @staticmethod
    def forward(ctx, x, weight, bias, store, layer, a_key, e_key):
        ctx.save_for_backward(x, weight)
        ctx.meta = (store, layer, e_key, bias is not None)
        if a_key is not None:
            store.put(layer, a_key, x.reshape(-1, x.shape[-1]))
        w = weight.to(x.dtype)
        return F.linear(x, w, None if bias is None else bias.to(x.dtype))

    @staticmethod
    def backward(ctx, gy):
        x, weight = ctx.saved_tensors
        store, layer, e_key, has_bias = ctx.meta
        g2 = gy.reshape(-1, gy.shape[-1])
        store.put(layer, e_key, g2)
        gx = gy @ weight.to(gy.dtype)
        gw = (g2.t() @ x.reshape(-1, x.shape[-1]).to(g2.dtype)).float()
        gb = g2.float().sum(0) if has_bias else None
        return gx, gw, gb, None, None, None, None


class EncoderLayer(nn.Module):
    def __init__(self, cfg: BertConfig, index: int, store: TapeStore):
        super().__init__()
        h, f = cfg.hidden, cfg.ffn
        self.cfg, self.index, self.store = cfg, index, store
        std = 0.02
        self.w = nn.ParameterDict({
            "q": nn.Parameter(torch.randn(h, h) * std), "k": nn.Parameter(torch.randn(h, h) * std),
            "v": nn.Parameter(torch.randn(h, h) * std), "o": nn.Parameter(torch.randn(h, h) * std),
            "ffn1": nn.Parameter(torch.randn(f, h) * std), "ffn2": nn.Parameter(torch.randn(h, f) * std)})
        self.b = nn.ParameterDict({k: nn.Parameter(torch.zeros(v.shape[0])) for k, v in self.w.items()})
        self.ln1 = nn.LayerNorm(h)
        self.ln2 = nn.LayerNorm(h)

    def lin(self, name: str, x, a_key: Optional[str]):
        return _TapedLinear.apply(x, self.w[name], self.b[name], self.store, self.index, a_key,
                                  "e_" + name)

    def forward(self, x):  # x: [B, S, h] (post-LN BERT)
        B, S, h = x.shape
        nh = self.cfg.heads
        q = self.lin("q", x, "a_qkv")
        k = self.lin("k", x, None)  # same input tape as q
        v = self.lin("v", x, None)
        split = lambda t: t.view(B, S, nh, h // nh).transpose(1, 2)  # noqa: E731
        ctx = F.scaled_dot_product_attention(split(q), split(k), split(v))
        ctx = ctx.transpose(1, 2).reshape(B, S, h)
        x = self.ln1(x + self.lin("o", ctx, "a_o"))
        y = F.gelu(self.lin("ffn1", x, "a_ffn1"))
        return self.ln2(x + self.lin("ffn2", y, "a_ffn2"))


class BertStage(nn.Module):
    """Encoder layers [first, first + count) (+ embeddings / MLM head)."""

    def __init__(self, cfg: BertConfig, first: int, count: int, is_first: bool, is_last: bool):
        super().__init__()
        self.cfg, self.first, self.count = cfg, first, count
        self.is_first, self.is_last = is_first, is_last
        self.store = TapeStore()
        self.layers = nn.ModuleList([EncoderLayer(cfg, i, self.store) for i in range(count)])
        if is_first:
            self.tok = nn.Embedding(cfg.vocab, cfg.hidden)
            self.pos = nn.Embedding(cfg.max_pos, cfg.hidden)
            self.ln_emb = nn.LayerNorm(cfg.hidden)
        if is_last:
            self.mlm_dense = nn.Linear(cfg.hidden, cfg.hidden)
            self.mlm_ln = nn.LayerNorm(cfg.hidden)
            self.decoder = nn.Linear(cfg.hidden, cfg.vocab)

    def kfac_layers(self) -> List[EncoderLayer]:
        return list(self.layers)

    def forward(self, x, mlm_positions=None, mlm_labels=None):
        """First stage: x = token ids [B, S]; others: hidden [B, S, h].
        Last stage returns the scalar MLM loss, others the hidden state."""
        # (no autocast weight cache: the stage may be captured into CUDA graphs)
        with torch.autocast("cuda", dtype=torch.bfloat16, enabled=x.is_cuda, cache_enabled=False):
            if self.is_first:
                pos = torch.arange(x.shape[1], device=x.device)
                x = self.ln_emb(self.tok(x) + self.pos(pos)[None])
            for layer in self.layers:
                x = layer(x)
            if not self.is_last:
                return x
            h = x.reshape(-1, x.shape[-1])[mlm_positions]
            h = self.mlm_ln(F.gelu(self.mlm_dense(h)))
            logits = self.decoder(h)
            return F.cross_entropy(logits.float(), mlm_labels)


def synthetic_batch(cfg: BertConfig, batch: int, seq: int, seed: int, device) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Token ids, flat MLM positions and labels (random init, no dataset:
    there is no network)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    ids = torch.randint(0, cfg.vocab, (batch, seq), generator=g)
    n_mask = max(1, int(math.ceil(cfg.mlm_fraction * batch * seq)))
    pos = torch.randperm(batch * seq, generator=g)[:n_mask].sort().values
    labels = torch.randint(0, cfg.vocab, (n_mask,), generator=g)
    return ids.to(device), pos.to(device), labels.to(device)
