"""Generate the rms_norm / fused_add_rms_norm kernel x model corpus entries
(BASELINE.json configs[4]): the config-1 port (workloads/rms_norm, Llama-2-7B
hidden 4096) and the Fig. 2 port (workloads/fused_add_rms_norm, hidden 7168)
under other models' hidden sizes -- the model-fixed tensor shapes of the
inferred context (row width of the two activations, weight length)
substituted.  Hidden sizes are the public HF configs; fused_add_rms_norm at
8192 is SPEC.md's section 2.3 variant.  Goldens come from the reference:
python oracle/gen_golden.py <base>_<model>.

    python tools/make_rms_variants.py [rms_norm|fused_add_rms_norm]"""
import copy
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MODELS = {
    "llama2_13b": 5120,
    "llama3_70b": 8192,
    "qwen2_7b": 3584,
    "gemma_7b": 3072,
    "deepseek_v3": 7168,
}

FUSED_MODELS = {
    "llama3_8b": 4096,
    "llama2_13b": 5120,
    "llama3_70b": 8192,
    "qwen2_7b": 3584,
}


def main(base_name="rms_norm"):
    BASE = os.path.join(ROOT, "workloads", base_name)
    models = MODELS if base_name == "rms_norm" else FUSED_MODELS
    ctx = json.load(open(os.path.join(BASE, "ctx.json")))
    for name, hidden in models.items():
        c = copy.deepcopy(ctx)
        for a in c["args"]:
            for k in a.get("constraints", []):
                if a["position"] in (0, 1) and k["feature"] == "dim1":
                    k["value"] = hidden
                if a["position"] in (0, 1) and k["feature"] == "numel":
                    k["coeff"] = hidden
                if a["position"] == 2 and k["feature"] in ("dim0", "numel"):
                    k["value"] = hidden
        d = os.path.join(ROOT, "workloads", f"{base_name}_{name}")
        os.makedirs(d, exist_ok=True)
        shutil.copy(os.path.join(BASE, "kernel.mk"), os.path.join(d, "kernel.mk"))
        with open(os.path.join(d, "ctx.json"), "w") as fh:
            json.dump(c, fh, indent=1)
        print(d)


if __name__ == "__main__":
    import sys

    main(sys.argv[1] if len(sys.argv) > 1 else "rms_norm")
