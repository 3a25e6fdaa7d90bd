"""Seeded synthetic-input generators shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no gather, reduce-scatter, Adam,
layer math or scheduling).  It only defines:

* the counter-based value generator (splitmix64 -> uniform with a given std),
  which the CUDA init kernel re-implements independently (init_param_kernel in
  paper_2504_09983_b200/csrc/glue.cu);
* the workload recipes: model shapes of the paper's workloads (§5.1,
  lines 440-444: Llama-3 / Mixtral shaped layers, bf16) and the parameter table
  order (first-use order of the S_0 rewrite, §4.1).
"""
from .gen import (splitmix64, uniform_u24, values, std_to_k, K_MLP, K_UNIT,
                  SEED_WEIGHTS, seed_inputs, seed_targets)
from .models import (ModelConfig, ParamSpec, llama_param_table, mlp_param_table, moe_param_table,
                     param_table, compute_ops, LLAMA3_8B, LLAMA3_70B, MIXTRAL_8X7B, small_llama,
                     small_mixtral, MLP_CONFIG1)

__all__ = [
    "splitmix64", "uniform_u24", "values", "std_to_k", "K_MLP", "K_UNIT",
    "SEED_WEIGHTS", "seed_inputs", "seed_targets",
    "ModelConfig", "ParamSpec", "llama_param_table", "mlp_param_table", "moe_param_table",
    "param_table", "compute_ops", "LLAMA3_8B", "LLAMA3_70B", "MIXTRAL_8X7B", "small_llama",
    "small_mixtral", "MLP_CONFIG1",
]
