"""NVLink evidence for the expert-parallel transport: a 2-rank
EP layer at the LongCat shape (8192 tokens per GPU).  Launch rank 0 under ncu
with NVLink metrics and rank 1 plainly:

    ncu --metrics nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum \
        -k regex:'ep_put_rows|grouped_gemm' --csv --log-file OUT python ep_nvlink_probe.py 0 &
    python ep_nvlink_probe.py 1

Prints this rank's expected peer payload (rows x 12 KB from the slot-count
matrix) so the ncu per-kernel NVLink bytes can be compared with it."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

rank, world = int(sys.argv[1]), 2
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29411")
torch.cuda.set_device(rank)
dist.init_process_group("gloo", rank=rank, world_size=world)
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id  # noqa: E402
from paper_2509_01322_b200.layer import LONGCAT  # noqa: E402

T, D = 8192, LONGCAT.d
ep = ExpertParallelLayer(P.Context(rank), LONGCAT, rank, world, 5, broadcast_unique_id(),
                         max_tokens=T)
a1 = torch.from_numpy(P.fill_normal(P.stream_seed(99, rank), T * D, threads=8)).cuda()
for _ in range(3):
    ep.forward(a1, None, None, T)
torch.cuda.synchronize()
ep.synchronize()
M = ep.count_matrix()
send, recv, own = int(M[rank].sum()), int(M[:, rank].sum()), int(M[rank, rank])
print(json.dumps({"rank": rank, "slot_matrix": M.tolist(),
                  "dispatch_tx_bytes": (send - own) * (D * 2 + 4),
                  "return_tx_bytes": (recv - own) * D * 2,
                  "note": "per layer call; ep_put_rows sends the dispatch rows (+ 4 B expert id), "
                          "GEMM2's epilogue sends the returned rows"}), flush=True)
dist.barrier()
ep.close()
dist.destroy_process_group()
