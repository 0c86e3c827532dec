"""Generate BASELINE.json configs[2] at its stated domain:
vLLM paged_attention v1 / v2, Mistral-7B (32 heads, 8 kv heads, head 128),
128 threads, symbolic seq_len up to 2^20 (the reference caps SL at 1e6,
context.py:508-524), a 2^20-block KV cache (block-table contents in
[0, 2^20 - 1]) and block_size in {8, 16, 32} (vLLM instantiates the kernel
per block size, so each is its own workload).

  paged_attention_v1_long_b{8,16,32}   v1 port of workloads/paged_attention_v1
  paged_attention_v2_long_b16          v2 port (512-token partitions) with
                                       max_num_seqs 1024: the partition
                                       scratch index
                                       ((seq * heads + head) * partitions
                                        + partition) * 128 + tid
                                       is i32 in vLLM and reaches
                                       1000 * 32 * 1954 * 128 > 2^31 at long
                                       context -- the paper's int32 hunt
                                       

The kernel text is the round-1 port with the block size substituted; the
contexts are the round-1 contexts with the long-context shapes.  Goldens:
python oracle/gen_golden.py <name>, then oracle/z3_crosscheck.py for the
sites the reference times out on."""
import copy
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W = os.path.join(ROOT, "workloads")

NUM_BLOCKS = 1 << 20
SEQ_MAX = 1 << 20


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


def _v1_kernel(bs: int) -> str:
    src = open(os.path.join(W, "paged_attention_v1", "kernel.mk")).read()
    head, body = src.split("\n", 1)
    body = (body.replace("+ 15) / 16) * 16", f"+ {bs - 1}) / {bs}) * {bs}")
                .replace("(seq_len + 15) / 16", f"(seq_len + {bs - 1}) / {bs}")
                .replace("lane % 16", f"lane % {bs}")
                .replace("block_idx * 16 + off", f"block_idx * {bs} + off")
                .replace("if (lane < 16)", f"if (lane < {min(bs, 32)})")
                .replace("i64(lane * 16)", f"i64(lane * {bs})"))
    return (f"# config 3 at its stated domain: vLLM paged_attention_v1_kernel, Mistral-7B (32 heads, "
            f"8 kv heads, head 128),\n# block {bs}, 128 threads, seq_len up to 2^20, 2^20-block KV cache "
            f"(tools/make_pa_long.py)\n" + body)


def _v2_kernel() -> str:
    src = open(os.path.join(W, "paged_attention_v2", "kernel.mk")).read()
    lines = [ln for ln in src.split("\n") if not ln.startswith("#")]
    return ("# config 3 at its stated domain: vLLM paged_attention_v2_kernel, Mistral-7B, block 16, "
            "512-token partitions,\n# seq_len up to 2^20, max_num_seqs 1024, 2^20-block KV cache "
            "(tools/make_pa_long.py)\n" + "\n".join(lines))


def make_v1(bs: int) -> None:
    ctx = json.load(open(os.path.join(W, "paged_attention_v1", "ctx.json")))
    args = {a["position"]: a for a in ctx["args"]}
    per_seq = SEQ_MAX // bs
    # key_cache [num_blocks, kv_heads, head/8, block, 8]; value_cache [num_blocks, kv_heads, head, block]
    _set(args[2], "dim0", NUM_BLOCKS)
    _set(args[2], "dim2", 16)
    _set(args[2], "dim3", bs)
    _set(args[2], "numel", NUM_BLOCKS * 8 * 16 * bs * 8)
    _set(args[3], "dim0", NUM_BLOCKS)
    _set(args[3], "dim3", bs)
    _set(args[3], "numel", NUM_BLOCKS * 8 * 128 * bs)
    _set(args[6], "dim1", per_seq)
    _set(args[6], "numel", per_seq)
    _set(args[6], "int_max", NUM_BLOCKS - 1)
    for grp in ctx["equal"]:
        # dim2 (head/8 = 16) and dim3 (block) are no longer one class for bs != 16
        if "arg2.dim2" in grp and bs != 16:
            grp[:] = ["arg2.dim2"]
        # the round-1 context had num_blocks == max_num_blocks_per_seq == 2048
        if "arg6.dim1" in grp:
            grp.remove("arg6.dim1")
    ctx["equal"] = [g for g in ctx["equal"] if len(g) > 1]
    if bs != 16:
        ctx["equal"].append(["arg2.dim3", "arg3.dim3"])
    ctx["globals"] = {"batch_size_max": 256, "seq_len_max": SEQ_MAX}
    name = f"paged_attention_v1_long_b{bs}"
    os.makedirs(os.path.join(W, name), exist_ok=True)
    with open(os.path.join(W, name, "ctx.json"), "w") as fh:
        json.dump(ctx, fh, indent=2)
    with open(os.path.join(W, name, "kernel.mk"), "w") as fh:
        fh.write(_v1_kernel(bs))


def make_v2() -> None:
    ctx = json.load(open(os.path.join(W, "paged_attention_v2", "ctx.json")))
    args = {a["position"]: a for a in ctx["args"]}
    seqs = 1000                      # max_num_seqs 1024, capped by the reference at 1000
    parts = -(-1000000 // 512)       # partitions at the reference's SL cap
    for p in (1, 2):                 # exp_sums, max_logits [seqs, heads, partitions]
        _set(args[p], "dim0", seqs)
        _set(args[p], "dim2", parts)
        _set(args[p], "numel", seqs * 32 * parts)
    _set(args[3], "dim0", seqs)      # tmp_out [seqs, heads, partitions, head]
    _set(args[3], "dim2", parts)
    _set(args[3], "numel", seqs * 32 * parts * 128)
    _set(args[5], "dim0", NUM_BLOCKS)
    _set(args[5], "numel", NUM_BLOCKS * 8 * 16 * 16 * 8)
    _set(args[6], "dim0", NUM_BLOCKS)
    _set(args[6], "numel", NUM_BLOCKS * 8 * 128 * 16)
    _set(args[9], "dim1", SEQ_MAX // 16)
    _set(args[9], "numel", SEQ_MAX // 16)
    _set(args[9], "int_max", NUM_BLOCKS - 1)
    for grp in ctx["equal"]:
        # the round-1 context had num_blocks == max_num_blocks_per_seq == 2048
        if "arg9.dim1" in grp:
            grp.remove("arg9.dim1")
    ctx["globals"] = {"batch_size_max": 1024, "seq_len_max": SEQ_MAX}
    name = "paged_attention_v2_long_b16"
    os.makedirs(os.path.join(W, name), exist_ok=True)
    with open(os.path.join(W, name, "ctx.json"), "w") as fh:
        json.dump(ctx, fh, indent=2)
    with open(os.path.join(W, name, "kernel.mk"), "w") as fh:
        fh.write(_v2_kernel())


def main():
    for bs in (8, 16, 32):
        make_v1(bs)
    make_v2()


if __name__ == "__main__":
    main()
