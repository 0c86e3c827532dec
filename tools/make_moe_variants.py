"""Generate the fused-MoE kernel x model corpus entries (BASELINE.json
configs[3]/[4]) from the Mixtral-8x7B ports under other MoE models' expert
count and top-k (public HF configs):

  moe_align_<model>    workloads/moe_align_mixtral: topk_ids row width and
                       element count (top-k), content bound (experts - 1), the
                       num_experts argument;
  topk_softmax_<model> workloads/topk_softmax: the three [T, top-k] outputs
                       (width, element count, index content bounds) and the
                       [T, experts] gating input.

Goldens come from the reference: python oracle/gen_golden.py <name>.

    python tools/make_moe_variants.py [moe_align|topk_softmax]"""
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


def topk_main():
    base = os.path.join(ROOT, "workloads", "topk_softmax")
    ctx = json.load(open(os.path.join(base, "ctx.json")))
    for name, (experts, topk) in MODELS.items():
        c = copy.deepcopy(ctx)
        for a in c["args"]:
            for k in a["constraints"]:
                if a["position"] in (0, 1, 2):
                    if k["feature"] == "dim1":
                        k["value"] = topk
                    elif k["feature"] == "numel":
                        k["coeff"] = topk
                    elif a["position"] == 1 and k["feature"] == "int_max":
                        k["value"] = experts - 1
                    elif a["position"] == 2 and k["feature"] == "int_max":
                        k["coeff"] = topk
                elif a["position"] == 3:
                    if k["feature"] == "dim1":
                        k["value"] = experts
                    elif k["feature"] == "numel":
                        k["coeff"] = experts
        d = os.path.join(ROOT, "workloads", f"topk_softmax_{name}")
        os.makedirs(d, exist_ok=True)
        shutil.copy(os.path.join(base, "kernel.mk"), os.path.join(d, "kernel.mk"))
        with open(os.path.join(d, "ctx.json"), "w") as fh:
            json.dump(c, fh, indent=1)
        print(d)


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
    import sys

    (topk_main if len(sys.argv) > 1 and sys.argv[1] == "topk_softmax" else main)()
