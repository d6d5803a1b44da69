"""Phase B "KVs Retrieve" timing (episodic.hpp:244-249, PAPER.md:455-465:
2.0-7.9 ms on A100 for Llama-3.2-3B at M = 2K..8K): an episode cache of the
Llama-3.2-3B shape (28 layers x 8 kv heads, d = 128, bf16) with M entries per
head, (a) held in pinned host memory and copied to HBM, (b) read back from
its .epkv file (the reference's fp64 format) through the GPU reader
(store.retrieve), (c) through the host-side parse (store.load_cache)."""
import json
import os
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_17396_b200 as epk  # noqa: E402

L, H, d = 28, 8, 128
out = {}
tmp = tempfile.mkdtemp()
for M in (2048, 4096, 6144, 8192):
    c = epk.EpisodeCache(L, H, d, [H * M] * L, torch.bfloat16, "cuda")
    c.set_regions(M)
    c.head_len.fill_(M)
    c.k.normal_()
    c.v.normal_()
    c.pos.copy_(torch.arange(H * M, device="cuda", dtype=torch.int32).repeat(L) % M)
    kv_bytes = 2 * c.k.numel() * 2
    hk, hv = torch.empty_like(c.k, device="cpu").pin_memory(), torch.empty_like(c.v, device="cpu").pin_memory()
    hk.copy_(c.k)
    hv.copy_(c.v)
    dst = epk.EpisodeCache(L, H, d, [H * M] * L, torch.bfloat16, "cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        dst.k.copy_(hk, non_blocking=True)
        dst.v.copy_(hv, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    path = os.path.join(tmp, f"ep_{M}.epkv")
    nbytes = epk.persist(c, path, episode_id=0, budget_per_head=M)
    epk.retrieve(path)
    torch.cuda.synchronize()
    t = time.perf_counter()
    epk.retrieve(path)
    torch.cuda.synchronize()
    t_dev = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    epk.load_cache(path, exact=False)
    torch.cuda.synchronize()
    t_host = (time.perf_counter() - t) * 1e3
    out[f"M={M}"] = {"kv_bytes_bf16": kv_bytes, "pinned_h2d_ms": best, "pinned_h2d_gbs": kv_bytes / best / 1e6,
                     "epkv_file_bytes": nbytes, "retrieve_gpu_reader_ms": t_dev, "load_cache_host_parse_ms": t_host}
    os.remove(path)
    del c, dst, hk, hv
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
