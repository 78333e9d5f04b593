"""The planner parity cases (shared by make_golden.py and the tests)."""


def dense_doc(N, K, eb, hi=8192):
    return {"name": "dense", "axes": [{"name": "i", "kind": "space", "range": [1, hi]},
                                      {"name": "j", "kind": "space", "extent": N},
                                      {"name": "k", "kind": "reduce", "extent": K}],
            "accesses": [{"tensor": "A", "axes": ["i", "k"], "role": "input"},
                         {"tensor": "B", "axes": ["k", "j"], "role": "input"},
                         {"tensor": "C", "axes": ["i", "j"], "role": "output"}],
            "elem_bytes": eb, "flops_per_point": 2}


def bmm_doc(b, i, j, k, eb=2):
    def ax(n, kind, v):
        return {"name": n, "kind": kind, **({"range": list(v)} if isinstance(v, tuple) else {"extent": v})}
    return {"name": "bmm", "axes": [ax("b", "space", b), ax("i", "space", i), ax("j", "space", j), ax("k", "reduce", k)],
            "accesses": [{"tensor": "A", "axes": ["b", "i", "k"], "role": "input"},
                         {"tensor": "B", "axes": ["b", "k", "j"], "role": "input"},
                         {"tensor": "C", "axes": ["b", "i", "j"], "role": "output"}],
            "elem_bytes": eb, "flops_per_point": 2}


def _c(cid, hw, doc, binding, legal=False, cap=1 << 21, topk_stream=False, big=False):
    return {"id": cid, "hw": hw, "doc": doc, "binding": binding, "legal": legal, "cap": cap,
            "topk_stream": topk_stream, "big": big}


CASES = [
    # C0: fp32 Dense N=K=768 on the FFMA descriptor
    *[_c(f"c0_m{m}", "b200_ffma", dense_doc(768, 768, 4, 512), {"i": m}) for m in (1, 2, 7, 53, 64, 127, 509, 512)],
    # C1/C3 Dense, bf16 descriptor, parity mode
    _c("c1_qkv_m160", "b200_bf16", dense_doc(2304, 768, 2), {"i": 160}),
    _c("c1_out_m1216", "b200_bf16", dense_doc(768, 768, 2), {"i": 1216}, topk_stream=True),
    _c("c3_m1", "b200_bf16", dense_doc(4096, 4096, 2), {"i": 1}),
    _c("c3_m16", "b200_bf16", dense_doc(4096, 4096, 2), {"i": 16}),
    _c("c3_m127", "b200_bf16", dense_doc(4096, 4096, 2), {"i": 127}, topk_stream=True),
    _c("c3_m1000", "b200_bf16", dense_doc(4096, 4096, 2), {"i": 1000}, topk_stream=True, big=True),
    # BMM (attention), parity mode
    _c("c1_scores_t5", "b200_bf16", bmm_doc(384, (1, 512), (1, 512), 64), {"i": 5, "j": 5}),
    _c("c1_scores_t38", "b200_bf16", bmm_doc(384, (1, 512), (1, 512), 64), {"i": 38, "j": 38}, topk_stream=True),
    _c("c1_context_t5", "b200_bf16", bmm_doc(384, (1, 512), 64, (1, 512)), {"i": 5, "k": 5}),
    _c("c2_scores_t1", "b200_bf16", bmm_doc(1024, (1, 512), (1, 512), 64), {"i": 1, "j": 1}),
    # B200 (tcgen05 legality) mode
    _c("b200_qkv_m160", "b200_bf16", dense_doc(2304, 768, 2), {"i": 160}, legal=True),
    _c("b200_qkv_m1216", "b200_bf16", dense_doc(2304, 768, 2), {"i": 1216}, legal=True),
    _c("b200_ffn1_m1984", "b200_bf16", dense_doc(3072, 768, 2), {"i": 1984}, legal=True),
    _c("b200_out_m4096", "b200_bf16", dense_doc(768, 768, 2), {"i": 4096}, legal=True),
    _c("b200_scores_t38", "b200_bf16", bmm_doc(384, (1, 512), (1, 512), 64), {"i": 38, "j": 38}, legal=True),
    _c("b200_context_t100", "b200_bf16", bmm_doc(384, (1, 512), 64, (1, 512)), {"i": 100, "k": 100}, legal=True),
    # V100-like descriptor (the paper's target) incl. a capped (truncated) enumeration
    _c("v100_m53", "v100_like", dense_doc(768, 768, 4, 128), {"i": 53}),
    _c("v100_m64_cap", "v100_like", dense_doc(768, 768, 4, 128), {"i": 64}, cap=40000),
    # big pools (5.9M-201M plans): Top-10 from the streaming
    # oracle of reference primitives only (the reference cannot materialise them)
    _c("c2_scores_t257", "b200_bf16", bmm_doc(1024, (1, 512), (1, 512), 64), {"i": 257, "j": 257}, topk_stream=True, big=True),
    _c("c2_scores_t512", "b200_bf16", bmm_doc(1024, (1, 512), (1, 512), 64), {"i": 512, "j": 512}, topk_stream=True, big=True),
    _c("c2_context_t512", "b200_bf16", bmm_doc(1024, (1, 512), 64, (1, 512)), {"i": 512, "k": 512}, topk_stream=True, big=True),
    _c("c3_m4096", "b200_bf16", dense_doc(4096, 4096, 2), {"i": 4096}, topk_stream=True, big=True),
    _c("c3_m8191", "b200_bf16", dense_doc(4096, 4096, 2), {"i": 8191}, topk_stream=True, big=True),
    _c("c1_ffn1_m1696", "b200_bf16", dense_doc(3072, 768, 2), {"i": 1696}, topk_stream=True, big=True),
    _c("c1_out_m1696", "b200_bf16", dense_doc(768, 768, 2), {"i": 1696}, topk_stream=True, big=True),
]
