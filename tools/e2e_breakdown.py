"""Where the e2e epoch time goes (C3): kernel time alone vs kernel time while the next
epoch's H2D copy (+ decode) runs on the copy stream, and the copy time alone."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11682_b200 import _native as nat, lsh, synth  # noqa: E402
from paper_2111_11682_b200.data import BaselineStats  # noqa: E402
from paper_2111_11682_b200.factorization import TrainConfig, init_params  # noqa: E402
from paper_2111_11682_b200.hogwild import HogwildTrainer  # noqa: E402
from paper_2111_11682_b200.similarity import NeighborTable  # noqa: E402

M, N, nnz, F, K, e = synth.SHAPES["c3"]
dm = synth.random_sparse_device(M, N, nnz, seed=0)
ent, _, _ = lsh.simlsh_topk_device(dm.dev, lsh.LshConfig(psi_exponent=e), K)
nbr = NeighborTable(N, K, nat.to_host(ent)[:N * K].reshape(N, K))
cfg = TrainConfig(F=F, K=K, epochs=20, seed=0)
stats = BaselineStats(dm.dev.mu, nat.to_host(dm.dev.base_b), nat.to_host(dm.dev.base_bhat))
tr = HogwildTrainer(None, nbr, cfg, dev=dm.dev, params=init_params(M, N, F, K, nbr, stats, cfg))
host = tr.pinned_stream()
bufs = tr._stream_buffers()
other = tuple(torch.empty_like(x) for x in bufs)
cs = torch.cuda.Stream()
comp = torch.cuda.current_stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


out = {}
for _ in range(2):
    tr.launch_epoch(0)
torch.cuda.synchronize()
# kernel alone
a, b = ev(), ev()
a.record()
for k in range(5):
    tr._launch_stream(bufs, k, tr.loss)
b.record()
torch.cuda.synchronize()
out["kernel_alone_ms"] = a.elapsed_time(b) / 5
# copy (+decode) alone
a, b = ev(), ev()
with torch.cuda.stream(cs):
    a.record(cs)
    for k in range(5):
        for dst, s_ in zip(other, host.values()):
            dst.copy_(s_, non_blocking=True)
    b.record(cs)
torch.cuda.synchronize()
out["copy_alone_ms"] = a.elapsed_time(b) / 5
a, b = ev(), ev()
a.record()
for k in range(5):
    tr._decode(other)
b.record()
torch.cuda.synchronize()
out["decode_alone_ms"] = a.elapsed_time(b) / 5
# kernel with a concurrent copy
ks = []
for k in range(5):
    a, b = ev(), ev()
    with torch.cuda.stream(cs):
        for dst, s_ in zip(other, host.values()):
            dst.copy_(s_, non_blocking=True)
    a.record()
    tr._launch_stream(bufs, k, tr.loss)
    b.record()
    torch.cuda.synchronize()
    ks.append(a.elapsed_time(b))
out["kernel_with_copy_ms"] = float(np.median(ks))
out["h2d_bytes"] = int(sum(v.numel() * v.element_size() for v in host.values()))
out["copy_gbs"] = out["h2d_bytes"] / out["copy_alone_ms"] / 1e6
# the e2e API itself
torch.cuda.synchronize()
t0 = time.perf_counter()
tr.train_from_host(host, 0, 10)
out["train_from_host_ms_per_epoch"] = (time.perf_counter() - t0) / 10 * 1e3
print(json.dumps(out), flush=True)
