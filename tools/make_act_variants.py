"""Kernel x model corpus for the narrowing-cast port (workloads/silu_and_mul,
vLLM act_and_mul_kernel): one workload per model's MLP intermediate size
(public HF configs), num_tokens in [1, 2^20].  Each has two sat narrowing
sites whose canonical witness is the first token count at which the int64
row offset no longer fits int32 (sat witnesses at scale for the device's
lexicographic reduction).  Goldens: python oracle/gen_golden.py silu_<model>."""
import copy
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = os.path.join(ROOT, "workloads", "silu_and_mul")

MODELS = {
    # name: MLP intermediate size
    "llama3_70b": 28672,
    "qwen2_7b": 18944,
    "gemma_7b": 24576,
    "mistral_7b": 14336,
    "llama2_13b": 13824,
    "deepseek_v2_lite": 10944,
}


def _set(arg, feature, value):
    for c in arg["constraints"]:
        if c["feature"] == feature:
            if c["law"] == "invariant":
                c["value"] = value
            elif c["law"] == "linear":
                c["coeff"] = value
            return
    raise KeyError(feature)


def main():
    base = json.load(open(os.path.join(BASE, "ctx.json")))
    for name, inter in MODELS.items():
        ctx = copy.deepcopy(base)
        args = {a["position"]: a for a in ctx["args"]}
        _set(args[0], "dim1", inter)
        _set(args[0], "numel", inter)
        _set(args[1], "dim1", 2 * inter)
        _set(args[1], "numel", 2 * inter)
        d = os.path.join(ROOT, "workloads", f"silu_{name}")
        os.makedirs(d, exist_ok=True)
        shutil.copy(os.path.join(BASE, "kernel.mk"), os.path.join(d, "kernel.mk"))
        with open(os.path.join(d, "ctx.json"), "w") as fh:
            json.dump(ctx, fh, indent=2)


if __name__ == "__main__":
    main()
