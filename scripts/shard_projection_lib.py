"""Shared helper of the shard projection scripts."""
import torch


def shard_kernel_ms(fn, g):
    """Per-shard device time of one iteration (its K2 + K3 + the shared
    combine), from CUPTI kernel records of a warm run (not replayed)."""
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    names = [e.name for e in ev]
    dur = [e.time_range.elapsed_us() / 1e3 for e in ev]
    # last iteration: the final combine and the g (K2, K3) pairs before it
    last = max(i for i, nm in enumerate(names) if "combine" in nm)
    k = [i for i in range(last) if "spmv_slot" in names[i] or "fixup" in names[i]][-2 * g:]
    comb = dur[last]
    return [dur[k[2 * r]] + dur[k[2 * r + 1]] + comb for r in range(g)]
