"""Generate the moe_align_block_size kernel x model corpus entries
(BASELINE.json configs[3]/[4]): the Mixtral-8x7B port (workloads/
moe_align_mixtral) under other MoE models' expert count and top-k (public HF
configs) -- the topk_ids row width and element count (top-k), its content
bound (experts - 1) and the num_experts argument substituted.  Goldens come
from the reference: python oracle/gen_golden.py moe_align_<model>."""
import copy
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = os.path.join(ROOT, "workloads", "moe_align_mixtral")

MODELS = {
    # name: (num_experts, top_k)
    "dbrx": (16, 4),
    "qwen15_moe": (60, 4),
    "deepseek_v2_lite": (64, 6),
    "arctic": (128, 2),
}


def main():
    ctx = json.load(open(os.path.join(BASE, "ctx.json")))
    for name, (experts, topk) in MODELS.items():
        c = copy.deepcopy(ctx)
        for a in c["args"]:
            for k in a["constraints"]:
                if a["position"] == 0 and k["feature"] == "dim1":
                    k["value"] = topk
                elif a["position"] == 0 and k["feature"] == "numel":
                    k["coeff"] = topk
                elif a["position"] == 0 and k["feature"] == "int_max":
                    k["value"] = experts - 1
                elif a["position"] == 1 and k["feature"] == "value":
                    k["value"] = experts
        d = os.path.join(ROOT, "workloads", f"moe_align_{name}")
        os.makedirs(d, exist_ok=True)
        shutil.copy(os.path.join(BASE, "kernel.mk"), os.path.join(d, "kernel.mk"))
        with open(os.path.join(d, "ctx.json"), "w") as fh:
            json.dump(c, fh, indent=1)
        print(d)


if __name__ == "__main__":
    main()
