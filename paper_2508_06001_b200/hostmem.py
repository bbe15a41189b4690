"""Page-locked host buffers for host<->device images (the e2e path)."""

_HOST_KEEP = []  # mmaps backing registered host buffers (alive for the process)
_CHOICE = {}     # per-process verdict of the upload probe: "thp" or "pinned"


def _thp_buffer(nbytes: int):
    """Anonymous mmap with MADV_HUGEPAGE, registered with cudaHostRegister (DMA
    over 2 MB pages when the kernel grants them); None if that fails."""
    import mmap

    import torch
    try:
        m = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        if hasattr(mmap, "MADV_HUGEPAGE"):
            m.madvise(mmap.MADV_HUGEPAGE)
        t = torch.frombuffer(m, dtype=torch.uint8)
        off = (-t.data_ptr()) % (2 << 20)
        t = t[off:off + nbytes]
        t.fill_(0)  # fault the pages in
        if int(torch.cuda.cudart().cudaHostRegister(t.data_ptr(), max(1, nbytes), 0)) != 0:
            return None
        _HOST_KEEP.append(m)
        return t
    except Exception:
        return None


def _upload_gbs(t, dev_buf) -> float:
    """H2D bandwidth of one buffer (best of 3 copies of up to 64 MB)."""
    import torch
    n = min(t.numel(), dev_buf.numel())
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev_buf[:n].copy_(t[:n], non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) * 1e6))
    return best


def _choose(nbytes: int) -> str:
    """Which allocator uploads faster on this box: the DMA rate of registered
    THP buffers and of cudaHostAlloc'd buffers each varied run to run (46-55
    GB/s, tools/upload_probe.py), so the first large request measures both."""
    import torch
    if "kind" in _CHOICE:
        return _CHOICE["kind"]
    n = min(nbytes, 64 << 20)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    thp = _thp_buffer(n)
    pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    g_pin = _upload_gbs(pin, dev)
    g_thp = _upload_gbs(thp, dev) if thp is not None else 0.0
    _CHOICE.update(kind="thp" if g_thp >= g_pin else "pinned", thp_gbs=g_thp, pinned_gbs=g_pin)
    return _CHOICE["kind"]


def choice() -> dict:
    """The probe's verdict ({} before the first large pinned_host call)."""
    return dict(_CHOICE)


def pinned_host(nbytes: int):
    """Page-locked host buffer for the e2e images: whichever of a registered
    THP mmap and torch's cudaHostAlloc'd allocator uploaded faster in this
    process's probe (buffers under 16 MB skip the probe: cudaHostAlloc)."""
    import torch
    if nbytes >= (16 << 20) and _choose(nbytes) == "thp":
        t = _thp_buffer(nbytes)
        if t is not None:
            return t
    return torch.empty(max(1, nbytes), dtype=torch.uint8, pin_memory=True)[:nbytes]
