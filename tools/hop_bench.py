"""Path-hop transport bandwidth between two GPUs (one process per GPU), the north_star's "P2P hops
as a fraction of NVLink bandwidth".

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/hop_bench.py

Rank 0 sends `reps` back-to-back messages of each size to rank 1 with
  * peer: spx_hop_push (SM stores into rank 1's CUDA-IPC-mapped buffer + release flag), per CTA
    count, rank 1 waiting on the flag with spx_hop_wait;
  * ce: spx_hop_push_ce (copy-engine memcpy into the mapped buffer + flag kernel), rank 1 waiting;
  * push_noflag / ce_noflag: the copy alone (SM stores / copy-engine cudaMemcpyAsync into the
    mapped peer buffer), no arrival flag;
  * nccl: torch.distributed send/recv on a two-rank NCCL communicator.
Times are CUDA events on rank 0's stream (the push / send side) and on rank 1's stream (the
receive side, from its first wait to its last); both reported.  One JSON line per point.
"""

from __future__ import annotations

import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2502_19913_b200 import native  # noqa: E402

NVLINK_GBS = 900.0


def main():
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    reps = 20
    sizes = [1 << 20, 8 << 20, 32 << 20, 128 << 20]
    big = torch.empty(max(sizes) // 2, dtype=torch.bfloat16, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    ex = {"buf": native.ipc_export(big), "flag": native.ipc_export(flags)}
    allx = [None, None]
    dist.all_gather_object(allx, ex)
    bases = {}

    def addr(hoff):
        h, off = hoff
        if h not in bases:
            bases[h] = native.ipc_open(h)
        return bases[h] + off

    lib = native.load()
    peer = allx[1 - rank]
    dst, flag = addr(peer["buf"]), addr(peer["flag"])
    s = torch.cuda.Stream(dev)
    expect = 0
    g = dist.new_group([0, 1])
    for nbytes in sizes:
        src = big[: nbytes // 2]
        for mode, ctas in [("peer", c) for c in (16, 32, 64, 128)] + [("ce", None), ("push_noflag", 32), ("ce_noflag", None), ("nccl", None)]:
            dist.barrier()
            for it in range(2):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(reps):
                    if mode == "ce_noflag":        # copy-engine memcpy into the mapped peer buffer
                        if rank == 0:
                            lib.spx_hop(local, ctypes.c_void_p(dst), local, ctypes.c_void_p(src.data_ptr()), nbytes,
                                        ctypes.c_void_p(s.cuda_stream))
                    elif mode == "push_noflag":    # the copy alone, no arrival flag
                        if rank == 0:
                            native.hop_push(dst, src, nbytes, 0, ctas, stream=s)
                    elif mode == "ce":             # the executor's default hop: CE copy + flag
                        if rank == 0:
                            native.hop_push_ce(dst, src, nbytes, flag, stream=s)
                        else:
                            expect += 1
                            native.hop_wait(flags, expect, stream=s)
                    elif mode == "peer":
                        if rank == 0:
                            native.hop_push(dst, src, nbytes, flag, ctas, stream=s)
                        else:
                            expect += ctas
                            native.hop_wait(flags, expect, stream=s)
                    else:
                        with torch.cuda.stream(s):
                            if rank == 0:
                                dist.send(src, 1, group=g)
                            else:
                                dist.recv(src, 0, group=g)
                e1.record(s)
                torch.cuda.synchronize(dev)
            us = torch.tensor([e0.elapsed_time(e1) * 1e3 / reps], device=dev)
            both = [torch.zeros(1, device=dev) for _ in range(2)]
            dist.all_gather(both, us)
            if rank == 0:
                us_s, us_r = float(both[0].item()), float(both[1].item())
                gbs = nbytes / (max(us_s, us_r) / 1e6) / 1e9
                print(json.dumps({"mode": mode, "ctas": ctas, "bytes": nbytes, "send_us": round(us_s, 2),
                                  "recv_us": round(us_r, 2), "gbs": round(gbs, 1),
                                  "frac_nvlink": round(gbs / NVLINK_GBS, 4)}), flush=True)
    torch.cuda.synchronize(dev)
    dist.barrier()
    for b in bases.values():
        native.ipc_close(b)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
