"""Synthetic shard workloads for the snapshot path.

A workload is a list of leaves (kind, path, size) in *creation/fill order* plus
the plan inputs (ModelSpec, ParallelTopology, rank) and a byte generator:

* ``mt19937_64``: one ``std::mt19937_64(seed)`` consumed leaf by leaf in spec
  order (reproduces the reference's golden C1 digests).
* ``splitmix64``: counter-based, word w of leaf i =
  mix64((seed ^ i*0xD1B54A32D192ED03) + (w+1)*0x9E3779B97F4A7C15), generated on
  the GPU by ``lzk_fill_splitmix`` and on the CPU by the oracle.

The spec text format is read by both the product tools and the oracle driver.
"""
from __future__ import annotations

import dataclasses
from typing import List, Tuple

__all__ = ["Workload", "gpt2_small", "llama7b_shard", "llama13b_shard", "llama70b_shard", "llama_layer_sample",
           "sweep_class", "dense_model_shard"]


@dataclasses.dataclass
class Workload:
    name: str
    param_count: int
    layer_count: int
    bpp_model: int
    bpp_opt: int
    leaves: List[Tuple[str, str, int]]  # (kind 'r'|'b', path, size) in fill order
    gen: str = "splitmix64"
    seed: int = 0
    topology: Tuple[int, int, int, int, int] = (1, 1, 1, 1, 1)
    rank: Tuple[int, int, int] = (0, 0, 0)
    step: int = 1

    @property
    def total_bytes(self) -> int:
        return sum(s for _, _, s in self.leaves)

    def spec_text(self) -> str:
        lines = [f"# lzk workload {self.name}",
                 f"model {self.param_count} {self.layer_count} {self.bpp_model} {self.bpp_opt}",
                 "topology " + " ".join(str(x) for x in self.topology),
                 "rank " + " ".join(str(x) for x in self.rank),
                 f"step {self.step}",
                 f"gen {self.gen} {self.seed}"]
        lines += [f"leaf {k} {p} {s}" for k, p, s in self.leaves]
        return "\n".join(lines) + "\n"

    def write_spec(self, path: str) -> str:
        with open(path, "w") as f:
            f.write(self.spec_text())
        return path


def _gpt2_small_tensors():
    d, ff, vocab, ctx = 768, 3072, 50257, 1024
    out = [("wte", vocab * d), ("wpe", ctx * d)]
    for l in range(12):
        p = f"h{l:02d}/"
        out += [(p + "ln_1.w", d), (p + "ln_1.b", d),
                (p + "attn.c_attn.w", d * 3 * d), (p + "attn.c_attn.b", 3 * d),
                (p + "attn.c_proj.w", d * d), (p + "attn.c_proj.b", d),
                (p + "ln_2.w", d), (p + "ln_2.b", d),
                (p + "mlp.c_fc.w", d * ff), (p + "mlp.c_fc.b", ff),
                (p + "mlp.c_proj.w", ff * d), (p + "mlp.c_proj.b", d)]
    out += [("ln_f.w", d), ("ln_f.b", d)]
    return out


def _model_state(name, tensors, bpp_model, layers, gen, seed):
    """params first (a_params/<t>, bpp_model*numel), then per tensor the fp32
    master + Adam m/v (b_optim/<t>/{fp32,exp_avg,exp_avg_sq}, 4*numel each)."""
    leaves = [("r", f"a_params/{n}", bpp_model * k) for n, k in tensors]
    for n, k in tensors:
        leaves += [("r", f"b_optim/{n}/fp32", 4 * k), ("r", f"b_optim/{n}/exp_avg", 4 * k),
                   ("r", f"b_optim/{n}/exp_avg_sq", 4 * k)]
    params = sum(k for _, k in tensors)
    return Workload(name, params, layers, bpp_model, 12, leaves, gen=gen, seed=seed)


def gpt2_small(seed: int = 125) -> Workload:
    """C1: GPT-2-small shard, 148 tensors, 124,439,808 params, 2+12 B/param,
    mt19937_64(125) fill."""
    return _model_state("c1-gpt2-small", _gpt2_small_tensors(), 2, 12, "mt19937_64", seed)


def _llama7b_tensors(layers=32, d=4096, ff=11008, vocab=32000):
    out = [("embed_tokens", vocab * d)]
    for l in range(layers):
        p = f"layers.{l:02d}/"
        out += [(p + "attn.q_proj", d * d), (p + "attn.k_proj", d * d),
                (p + "attn.v_proj", d * d), (p + "attn.o_proj", d * d),
                (p + "mlp.gate_proj", d * ff), (p + "mlp.up_proj", d * ff),
                (p + "mlp.down_proj", ff * d),
                (p + "input_norm", d), (p + "post_attn_norm", d)]
    out += [("norm", d), ("lm_head", vocab * d)]
    return out


def llama7b_shard(seed: int = 7, layers: int = 32, vocab: int = 32000, dp: int = 1, rank: int = 0,
                  name: str = "c2-llama7b") -> Workload:
    """C2: LLaMA-2-7B-shaped shard on one rank, 4+12 B/param (~107.8 GB).

    dp > 1 gives weak scaling: the plan is for a dp-times larger model, so
    every rank owns exactly one C2-sized shard (files layers-*/optimizer-<rank>)."""
    w = _model_state(name, _llama7b_tensors(layers=layers, vocab=vocab), 4, layers, "splitmix64", seed + rank)
    if dp > 1:
        w.param_count *= dp
        w.topology = (dp, 1, 1, dp, 1)
        w.rank = (rank, 0, 0)
    return w


def llama13b_shard(seed: int = 13, layers: int = 5, dp: int = 8, rank: int = 0,
                   name: str = "c3-llama13b") -> Workload:
    """C3 (BASELINE.json configs[2]): one rank's shard of a LLaMA-13B-shaped
    model (d=5120, ffn 13824, vocab 32000, 40 layers) over dp=8: 5 decoder
    layers plus embeddings, 4+12 B/param, ~26 GB per GPU."""
    w = _model_state(name, _llama7b_tensors(layers=layers, d=5120, ff=13824), 4, layers, "splitmix64", seed + rank)
    w.param_count *= dp
    w.topology = (dp, 1, 1, dp, 1)
    w.rank = (rank, 0, 0)
    return w


def _llama70b_tensors(layers=80, d=8192, kv=1024, ff=28672, vocab=32000):
    out = [("embed_tokens", vocab * d)]
    for l in range(layers):
        p = f"layers.{l:02d}/"
        out += [(p + "attn.q_proj", d * d), (p + "attn.k_proj", d * kv),
                (p + "attn.v_proj", d * kv), (p + "attn.o_proj", d * d),
                (p + "mlp.gate_proj", d * ff), (p + "mlp.up_proj", d * ff),
                (p + "mlp.down_proj", ff * d),
                (p + "input_norm", d), (p + "post_attn_norm", d)]
    out += [("norm", d), ("lm_head", vocab * d)]
    return out


def llama70b_shard(seed: int = 70, layers: int = 10, dp: int = 8, rank: int = 0,
                   name: str = "c4-llama70b") -> Workload:
    """C4 (BASELINE.json configs[3]): one rank's ZeRO-style shard of a
    LLaMA-2-70B-shaped model (d=8192, GQA k/v 8192x1024, ffn 28672, vocab
    32000) over dp=8: 80/8 = 10 decoder layers plus embeddings, 4+12 B/param,
    ~145 GB per GPU -- larger than any host pool it streams through."""
    w = _model_state(name, _llama70b_tensors(layers=layers), 4, layers, "splitmix64", seed + rank)
    w.param_count *= dp
    w.topology = (dp, 1, 1, dp, 1)
    w.rank = (rank, 0, 0)
    return w


def llama_layer_sample(seed: int = 7, layers: int = 1, dp: int = 1, rank: int = 0) -> Workload:
    """Bounded sample of C2 for the reference arm and the matched pair:
    `layers` LLaMA-7B decoder layers with the C2 tensor shapes and 4+12
    B/param (3.24 GB per layer). dp > 1: weak scaling, one such shard per rank."""
    tensors = [t for t in _llama7b_tensors(layers=layers) if t[0].startswith("layers.")]
    w = _model_state(f"c2-sample-{layers}l", tensors, 4, layers, "splitmix64", seed + rank)
    if dp > 1:
        w.param_count *= dp
        w.topology = (dp, 1, 1, dp, 1)
        w.rank = (rank, 0, 0)
    return w


def dense_model_shard(name: str, tensors, bpp_model: int, layers: int, seed: int) -> Workload:
    return _model_state(name, tensors, bpp_model, layers, "splitmix64", seed)


def sweep_class(tensor_bytes: int, total_bytes: int, seed: int = 5) -> Workload:
    """C5: one size class. A 1-layer model whose layer shard is one region and
    whose optimizer shard is split into equal tensors of ``tensor_bytes``."""
    n = max(1, total_bytes // tensor_bytes)
    opt = n * tensor_bytes
    # 2+12 B/param: pick params so that optimizer bytes == opt exactly
    params = opt // 12
    opt = params * 12
    leaves = [("r", "a/w", 2 * params)]
    sizes = [tensor_bytes] * (opt // tensor_bytes)
    rem = opt - sum(sizes)
    if rem:
        sizes.append(rem)
    leaves += [("r", f"b/t{i:07d}", s) for i, s in enumerate(sizes)]
    return Workload(f"c5-sweep-{tensor_bytes}", params, 1, 2, 12, leaves, gen="splitmix64", seed=seed)
