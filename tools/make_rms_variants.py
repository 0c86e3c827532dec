"""Generate the rms_norm kernel x model corpus entries (BASELINE.json
configs[4]): the config-1 port (workloads/rms_norm, Llama-2-7B hidden 4096)
under other models' hidden sizes -- the model-fixed tensor shapes of the
inferred context (input / out row width, weight length) substituted.
Hidden sizes are the public HF configs.  Goldens come from the reference:
python oracle/gen_golden.py rms_norm_<model>."""
import copy
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = os.path.join(ROOT, "workloads", "rms_norm")

MODELS = {
    "llama2_13b": 5120,
    "llama3_70b": 8192,
    "qwen2_7b": 3584,
    "gemma_7b": 3072,
    "deepseek_v3": 7168,
}


def main():
    ctx = json.load(open(os.path.join(BASE, "ctx.json")))
    for name, hidden in MODELS.items():
        c = copy.deepcopy(ctx)
        for a in c["args"]:
            for k in a.get("constraints", []):
                if a["position"] in (0, 1) and k["feature"] == "dim1":
                    k["value"] = hidden
                if a["position"] in (0, 1) and k["feature"] == "numel":
                    k["coeff"] = hidden
                if a["position"] == 2 and k["feature"] in ("dim0", "numel"):
                    k["value"] = hidden
        d = os.path.join(ROOT, "workloads", f"rms_norm_{name}")
        os.makedirs(d, exist_ok=True)
        shutil.copy(os.path.join(BASE, "kernel.mk"), os.path.join(d, "kernel.mk"))
        with open(os.path.join(d, "ctx.json"), "w") as fh:
            json.dump(c, fh, indent=1)
        print(d)


if __name__ == "__main__":
    main()
