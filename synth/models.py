"""Workload recipes: the shapes of the paper's models as synthetic layer stacks.

PAPER.md §5.1 (lines 440-444) evaluates Llama-3 70B and Mixtral 8x7B in bf16
with fp32 copies of params, grads and Adam states; BASELINE.json's configs add a
Llama-3 8B-shaped stack and the 4-layer MLP of config 1.  The synthetic layer
keeps the 7 Llama projections at their real shapes; the attention core is a
token-local surrogate.

The parameter table is listed in first-use order of the forward pass, which is
the order the fully-sharded rewrite gathers them in (§4.1).
The compute-op graph (which op consumes which parameter) is also defined here:
it is the workload's structure, not the method.
"""
from dataclasses import dataclass
from typing import List, Tuple

from .gen import std_to_k, K_MLP

WEIGHT_STD = 0.02


@dataclass(frozen=True)
class ModelConfig:
    name: str
    kind: str            # "llama" | "mlp"
    hidden: int
    ffn: int
    n_heads: int
    n_kv: int
    head_dim: int
    layers: int
    seq: int = 2048
    batch: int = 1
    n_experts: int = 0   # > 0: Mixtral-shaped MoE MLP (fixed balanced top-2 routing)

    @property
    def tokens(self) -> int:
        return self.seq * self.batch

    @property
    def q_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv * self.head_dim


@dataclass(frozen=True)
class ParamSpec:
    id: int              # global id == generator tensor_id == S_0 first-use order
    layer: int
    name: str
    shape: Tuple[int, ...]
    k: float             # generator scale; 0.0 means "constant 1.0" (norm gain)
    dtype: str           # "bf16" | "fp32"

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4


LLAMA_NAMES = ("attn_norm", "wq", "wk", "wv", "wo", "mlp_norm", "wgate", "wup", "wdown")


def llama_param_table(cfg: ModelConfig) -> List[ParamSpec]:
    kw = float(std_to_k(WEIGHT_STD))
    h, f, qd, kvd = cfg.hidden, cfg.ffn, cfg.q_dim, cfg.kv_dim
    shapes = {
        "attn_norm": (h,), "wq": (qd, h), "wk": (kvd, h), "wv": (kvd, h),
        "wo": (h, qd), "mlp_norm": (h,), "wgate": (f, h), "wup": (f, h),
        "wdown": (h, f),
    }
    out = []
    for l in range(cfg.layers):
        for j, nm in enumerate(LLAMA_NAMES):
            out.append(ParamSpec(id=l * len(LLAMA_NAMES) + j, layer=l, name=nm,
                                 shape=shapes[nm],
                                 k=0.0 if nm.endswith("norm") else kw,
                                 dtype="bf16"))
    return out


MOE_ATTN_NAMES = ("attn_norm", "wq", "wk", "wv", "wo", "mlp_norm", "router")


def moe_names(n_experts: int) -> Tuple[str, ...]:
    """Per-layer tensor names of the Mixtral-shaped layer in first-use order:
    attention, router, then each expert's w1 | w3 (gate | up) and w2 (down)."""
    out = list(MOE_ATTN_NAMES)
    for e in range(n_experts):
        out += ["w1_%d" % e, "w3_%d" % e, "w2_%d" % e]
    return tuple(out)


def moe_param_table(cfg: ModelConfig) -> List[ParamSpec]:
    """Mixtral 8x7B-shaped layer: 7 + 3 E tensors
    (31 at E = 8), router [E, h], experts w1, w3 [f, h] and w2 [h, f]."""
    kw = float(std_to_k(WEIGHT_STD))
    h, f, qd, kvd, E = cfg.hidden, cfg.ffn, cfg.q_dim, cfg.kv_dim, cfg.n_experts
    names = moe_names(E)
    out = []
    for l in range(cfg.layers):
        for j, nm in enumerate(names):
            base = nm.split("_")[0] if nm[0] == "w" and "_" in nm and nm[1].isdigit() else nm
            shape = {"attn_norm": (h,), "wq": (qd, h), "wk": (kvd, h), "wv": (kvd, h), "wo": (h, qd),
                     "mlp_norm": (h,), "router": (E, h), "w1": (f, h), "w3": (f, h), "w2": (h, f)}[base]
            out.append(ParamSpec(id=l * len(names) + j, layer=l, name=nm, shape=shape,
                                 k=0.0 if nm.endswith("norm") else kw, dtype="bf16"))
    return out


def param_table(cfg: ModelConfig) -> List[ParamSpec]:
    if cfg.kind == "mlp":
        return mlp_param_table(cfg)
    return moe_param_table(cfg) if cfg.n_experts else llama_param_table(cfg)


def mlp_param_table(cfg: ModelConfig) -> List[ParamSpec]:
    """Config 1: Linear(256,256)+bias x4, fp32, PyTorch-default U(+-1/16) init."""
    out = []
    for l in range(cfg.layers):
        out.append(ParamSpec(2 * l, l, "w", (cfg.hidden, cfg.hidden), float(K_MLP), "fp32"))
        out.append(ParamSpec(2 * l + 1, l, "b", (cfg.hidden,), float(K_MLP), "fp32"))
    return out


# --- compute-op graph -------------------------------------------------------
# Each op: dict(name, kind in {"compute","rs"}, phase in {"fwd","bwd"}, micro,
# layer, params=[param ids consumed]).  RS(l) is the reduce-scatter (+ Adam on
# the last micro-step) of layer l, placed after the layer's last backward op
# of every micro-step.

LLAMA_FWD = (("attn_norm", ("attn_norm",)), ("qkv", ("wq", "wk", "wv")),
             ("attn_mix", ()), ("o_proj", ("wo",)), ("mlp_norm", ("mlp_norm",)),
             ("gate_up", ("wgate", "wup")), ("act", ()), ("down", ("wdown",)))
LLAMA_BWD = (("down_bwd", ("wdown",)), ("act_bwd", ()), ("gate_up_bwd", ("wgate", "wup")),
             ("mlp_norm_bwd", ("mlp_norm",)), ("o_bwd", ("wo",)), ("attn_mix_bwd", ()),
             ("qkv_bwd", ("wq", "wk", "wv")), ("attn_norm_bwd", ("attn_norm",)))


# Layer-level activation checkpointing ("recomputing each
# layer as a block"): the forward keeps only each layer's output; the backward
# of layer l first re-runs the forward ops its gradients need (all but `down`).
LLAMA_RECOMPUTE = tuple(("re_" + nm, ps) for nm, ps in LLAMA_FWD if nm != "down")


def llama_compute_ops(cfg: ModelConfig, micro_steps: int = 1, checkpoint: bool = False):
    P = len(LLAMA_NAMES)
    pid = lambda l, nm: l * P + LLAMA_NAMES.index(nm)
    ops = []
    for mu in range(micro_steps):
        for l in range(cfg.layers):
            for nm, ps in LLAMA_FWD:
                ops.append(dict(name=nm, kind="compute", phase="fwd", micro=mu, layer=l,
                                params=[pid(l, p) for p in ps]))
        ops.append(dict(name="loss", kind="compute", phase="fwd", micro=mu,
                        layer=cfg.layers - 1, params=[]))
        for l in reversed(range(cfg.layers)):
            for nm, ps in (LLAMA_RECOMPUTE if checkpoint else ()) + LLAMA_BWD:
                ops.append(dict(name=nm, kind="compute", phase="bwd", micro=mu, layer=l,
                                params=[pid(l, p) for p in ps]))
            # every micro-step reduce-scatters into the partitioned fp32
            # accumulator; the last one also applies Adam
            ops.append(dict(name="rs", kind="rs", phase="bwd", micro=mu, layer=l, params=[]))
    return ops


def moe_compute_ops(cfg: ModelConfig, micro_steps: int = 1, checkpoint: bool = False):
    """Mixtral-shaped layer: the Llama attention ops, then router, token gather,
    per expert (gate|up GEMM, activation, down GEMM) and the gated combine.
    Backward mirrors it; the router backward also forms dL/dh2."""
    names = moe_names(cfg.n_experts)
    P = len(names)
    pid = lambda l, nm: l * P + names.index(nm)
    E = cfg.n_experts
    attn_f = LLAMA_FWD[:5]                                   # attn_norm .. mlp_norm
    mlp_f = [("router", ("router",)), ("moe_gather", ())]
    for e in range(E):
        mlp_f += [("exp_gu_%d" % e, ("w1_%d" % e, "w3_%d" % e)), ("exp_act_%d" % e, ()),
                  ("exp_down_%d" % e, ("w2_%d" % e,))]
    mlp_f += [("moe_combine", ())]
    mlp_b = [("moe_combine_bwd", ())]
    for e in range(E):
        mlp_b += [("exp_down_bwd_%d" % e, ("w2_%d" % e,)), ("exp_act_bwd_%d" % e, ()),
                  ("exp_gu_bwd_%d" % e, ("w1_%d" % e, "w3_%d" % e))]
    mlp_b += [("router_bwd", ("router",))]
    attn_b = LLAMA_BWD[3:]                                   # mlp_norm_bwd .. attn_norm_bwd
    fwd = tuple(attn_f) + tuple(mlp_f)
    # the combine's backward needs every expert output, so only the combine
    # itself is not re-run
    recompute = tuple(("re_" + nm, ps) for nm, ps in fwd if nm != "moe_combine")
    ops = []
    for mu in range(micro_steps):
        for l in range(cfg.layers):
            for nm, ps in fwd:
                ops.append(dict(name=nm, kind="compute", phase="fwd", micro=mu, layer=l,
                                params=[pid(l, p) for p in ps]))
        ops.append(dict(name="loss", kind="compute", phase="fwd", micro=mu, layer=cfg.layers - 1, params=[]))
        for l in reversed(range(cfg.layers)):
            for nm, ps in (recompute if checkpoint else ()) + tuple(mlp_b) + tuple(attn_b):
                ops.append(dict(name=nm, kind="compute", phase="bwd", micro=mu, layer=l,
                                params=[pid(l, p) for p in ps]))
            ops.append(dict(name="rs", kind="rs", phase="bwd", micro=mu, layer=l, params=[]))
    return ops


def compute_ops(cfg: ModelConfig, micro_steps: int = 1, checkpoint: bool = False):
    if cfg.n_experts:
        return moe_compute_ops(cfg, micro_steps, checkpoint)
    return llama_compute_ops(cfg, micro_steps, checkpoint)


LLAMA3_8B = ModelConfig("llama3-8b", "llama", 4096, 14336, 32, 8, 128, 32)
LLAMA3_70B = ModelConfig("llama3-70b", "llama", 8192, 28672, 64, 8, 128, 80)
# Mixtral 8x7B: Llama attention shapes, MoE MLP of 8 experts (f 14336) with
# fixed balanced top-2 routing
MIXTRAL_8X7B = ModelConfig("mixtral-8x7b", "llama", 4096, 14336, 32, 8, 128, 32, n_experts=8)
MLP_CONFIG1 = ModelConfig("mlp4x256", "mlp", 256, 256, 1, 1, 256, 4, seq=1, batch=8)


def small_llama(layers: int = 2, seq: int = 256, batch: int = 1) -> ModelConfig:
    """Scaled-down Llama layer for oracle-speed parity: same structure, GQA 2:1."""
    return ModelConfig("llama-small", "llama", 512, 1024, 4, 2, 128, layers, seq=seq, batch=batch)


def small_mixtral(layers: int = 2, seq: int = 256, batch: int = 1) -> ModelConfig:
    """Scaled-down Mixtral layer: 8 experts of f = 256, top-2 fixed routing."""
    return ModelConfig("mixtral-small", "llama", 512, 256, 4, 2, 128, layers, seq=seq, batch=batch, n_experts=8)
