"""Generate the kernel x model corpus (BASELINE.json configs[4]) for the
rotary-embedding port: one workload per model configuration, same kernel
port, model-fixed tensor shapes substituted into the inferred context of
workloads/rotary_embedding (Llama-3-8B).

    num_heads x head_size      query row width   (arg1.dim1)
    num_kv_heads x head_size   key row width     (arg2.dim1)
    max_position x rot_dim     cos_sin_cache     (arg4)
    head_size                  scalar argument   (arg3)

Model shapes are the public HF configs (NeoX-style rotary, rot_dim =
head_size).  Goldens come from the reference: python oracle/gen_golden.py
rotary_<model>."""
import copy
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = os.path.join(ROOT, "workloads", "rotary_embedding")

MODELS = {
    # name: (num_heads, num_kv_heads, head_size, max_position)
    "llama2_7b": (32, 32, 128, 4096),
    "mistral_7b": (32, 8, 128, 32768),
    "llama3_70b": (64, 8, 128, 8192),
    "qwen2_7b": (28, 4, 128, 32768),
    "llama2_13b": (40, 40, 128, 4096),
    "mixtral_8x7b": (32, 8, 128, 32768),
    "gemma_7b": (16, 16, 256, 8192),
}


def _set(arg, feature, value):
    for c in arg["constraints"]:
        if c["feature"] == feature:
            if c["law"] == "invariant":
                c["value"] = value
            elif c["law"] == "linear":
                c["coeff"] = value
            elif c["law"] == "upper_bound":
                c["max"] = value
            return
    raise KeyError(feature)


def main():
    base = json.load(open(os.path.join(BASE, "ctx.json")))
    src = open(os.path.join(BASE, "kernel.mk")).read()
    for name, (nh, nkv, hs, maxpos) in MODELS.items():
        ctx = copy.deepcopy(base)
        args = {a["position"]: a for a in ctx["args"]}
        _set(args[0], "int_max", maxpos - 1)
        _set(args[1], "dim1", nh * hs)
        _set(args[1], "numel", nh * hs)
        _set(args[2], "dim1", nkv * hs)
        _set(args[2], "numel", nkv * hs)
        _set(args[3], "value", hs)
        _set(args[4], "dim0", maxpos)
        _set(args[4], "dim1", hs)
        _set(args[4], "numel", maxpos * hs)
        out = os.path.join(ROOT, "workloads", f"rotary_{name}")
        os.makedirs(out, exist_ok=True)
        header = (f"# config 5 corpus: vLLM rotary_embedding_kernel (NeoX), {name}: {nh} q heads, "
                  f"{nkv} kv heads, head_size {hs}, max_position {maxpos}\n")
        body = src.split("\n", 1)[1] if src.startswith("#") else src
        open(os.path.join(out, "kernel.mk"), "w").write(header + body)
        json.dump(ctx, open(os.path.join(out, "ctx.json"), "w"), indent=2)
        print(out)


if __name__ == "__main__":
    main()
