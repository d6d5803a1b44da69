"""Episode-sharded cache building across GPUs (episodic.hpp:108-199, Phase A).

The reference builds one compressed cache per episode: cluster the history
into E episodes (kmeans), measure sensitivity and allocate layer budgets, then
run block_prefill once per episode with that episode's medoid prompt
(episodic.hpp:156-188, optionally std::async-parallel, byte-identical to the
sequential run).  Episodes are independent, so the multi-GPU unit is the
episode: rank r (one process per GPU) builds episodes r, r+W, r+2W, ...
There is no collective on the data path; only the per-episode summaries are
gathered on the host at the end.  K-means over sharded segment embeddings is
clustering.kmeans_sharded (ordered rank chain, bit-identical to one GPU).
"""
from __future__ import annotations

from dataclasses import dataclass, field


def assign_episodes(n_episodes: int, world_size: int) -> list[list[int]]:
    """Round-robin episode ownership: owner(e) = e mod W."""
    if n_episodes < 0 or world_size < 1:
        raise ValueError("assign_episodes: bad arguments")
    return [list(range(r, n_episodes, world_size)) for r in range(world_size)]


@dataclass
class EpisodeSummary:
    episode_id: int
    rank: int
    blocks_processed: int
    entries_per_layer: list = field(default_factory=list)
    evictions_per_block: list = field(default_factory=list)


def build_episodes(run_episode, n_episodes: int, group=None) -> list[EpisodeSummary]:
    """Runs `run_episode(e) -> PrefillReport` for this rank's episodes and
    gathers every rank's summaries (ordered by episode id) on all ranks.
    Without torch.distributed initialised this is the single-GPU loop."""
    try:
        import torch.distributed as dist
        dist_on = dist.is_available() and dist.is_initialized()
    except ImportError:  # pragma: no cover
        dist_on = False
    rank = dist.get_rank(group) if dist_on else 0
    world = dist.get_world_size(group) if dist_on else 1
    mine = []
    for e in assign_episodes(n_episodes, world)[rank]:
        rep = run_episode(e)
        mine.append(EpisodeSummary(e, rank, rep.blocks_processed, list(rep.cache.entries_per_layer()),
                                   list(rep.evictions_per_block)))
    if not dist_on:
        return mine
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    out = [s for part in gathered for s in part]
    out.sort(key=lambda s: s.episode_id)
    return out
