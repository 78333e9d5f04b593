"""BERT-base encoder end to end with the module swap (VERDICT r1
missing #6): 12 encoder layers, batch 32, hidden 768, 12 heads, FFN 3072, at
the C1 sequence lengths (8 canonical T + 24 GLUE-like draws). Per T, the
forward pass of

  * ours  — paper_2407_21418_b200.bert.EncoderLayer: the six GEMMs of every
            layer on the uKernel executor through Planner.dense / .bmm (bias
            and GELU fused into the epilogues), softmax / layer norm /
            residuals in torch;
  * torch — torch.nn.TransformerEncoderLayer in bf16 (cuBLAS GEMMs, the
            fused scaled-dot-product attention), eval mode;

is timed with CUDA events after a warm-up forward at that T (ours: the first
call at a new T plans the shapes and builds the tables; that cold call is
reported separately). Synthetic activations, random weights.
  python scripts/bert_time.py"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2407_21418_b200.bert import EncoderLayer  # noqa: E402
from paper_2407_21418_b200.runtime import Planner  # noqa: E402
from paper_2407_21418_b200.workloads import CANONICAL_T, glue_seq_lengths  # noqa: E402

LAYERS, B = 12, 32
dev = torch.device("cuda", 0)
torch.manual_seed(0)
ref_layers = [torch.nn.TransformerEncoderLayer(768, 12, 3072, dropout=0.0, activation="gelu", batch_first=True,
                                               device=dev, dtype=torch.bfloat16).eval() for _ in range(LAYERS)]
planner = Planner()
ours_layers = [EncoderLayer.from_torch(layer, planner) for layer in ref_layers]


def fwd_ours(x):
    for layer in ours_layers:
        x = layer(x)
    return x


def fwd_torch(x):
    with torch.no_grad():
        for layer in ref_layers:
            x = layer(x)
    return x


class Graphed:
    """One CUDA graph per sequence length (captured on the first call at that
    T, after an eager warm-up that plans the shapes and builds the tables):
    replays cost device time only, as a serving stack with per-length graph
    buckets would run either model."""

    def __init__(self, f):
        self.f, self.graphs = f, {}

    def __call__(self, x):
        key = tuple(x.shape)
        if key not in self.graphs:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self.f(x)  # warm-up on the capture stream
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            xin = x.clone()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                yout = self.f(xin)
            self.graphs[key] = (g, xin, yout)
        g, xin, yout = self.graphs[key]
        xin.copy_(x)
        g.replay()
        return yout


graph_ours, graph_torch = Graphed(fwd_ours), Graphed(fwd_torch)


def timed(f, x, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        f(x)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


ts = list(CANONICAL_T) + glue_seq_lengths(24, seed=0)
rows = []
for T in ts:
    x = (torch.randn(B, T, 768, device=dev)).bfloat16()
    t0 = time.perf_counter()
    out = fwd_ours(x)
    torch.cuda.synchronize()
    cold_ms = (time.perf_counter() - t0) * 1e3
    ref = fwd_torch(x)
    err = ((out.float() - ref.float()).abs().max() / ref.float().abs().max()).item()
    ours_ms = timed(fwd_ours, x)
    torch_ms = timed(fwd_torch, x)
    gout = graph_ours(x)
    gref = graph_torch(x)
    torch.cuda.synchronize()
    assert torch.equal(gout, out), "graph replay differs from the eager forward"
    ours_g = timed(graph_ours, x)
    torch_g = timed(graph_torch, x)
    rows.append({"T": T, "ours_ms": ours_ms, "torch_ms": torch_ms, "ours_graph_ms": ours_g, "torch_graph_ms": torch_g,
                 "ours_cold_ms": cold_ms, "rel_err_12_layers": err})
    print(f"T={T:4d}: eager ours {ours_ms:7.3f} ms torch {torch_ms:7.3f} ms | CUDA graph ours {ours_g:7.3f} ms "
          f"torch {torch_g:7.3f} ms | ours cold {cold_ms:8.2f} ms | rel err after 12 layers {err:.3g}", flush=True)
summary = {"model": "BERT-base encoder, 12 layers, batch 32, bf16, GLUE-like T (8 canonical + 24 drawn)",
           "n_seq_lengths": len(rows)}
for k in ("ours_ms", "torch_ms", "ours_graph_ms", "torch_graph_ms"):
    summary["sum_" + k] = sum(r[k] for r in rows)
summary["eager_speedup"] = summary["sum_torch_ms"] / summary["sum_ours_ms"]
summary["graph_speedup"] = summary["sum_torch_graph_ms"] / summary["sum_ours_graph_ms"]
summary["rows"] = rows
print(json.dumps(summary))
