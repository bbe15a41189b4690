"""Page-locked host buffers for host<->device images (the e2e path)."""

_HOST_KEEP = []  # mmaps backing registered host buffers (alive for the process)


def pinned_host(nbytes: int):
    """Page-locked host buffer for the e2e images: anonymous mmap with
    MADV_HUGEPAGE, registered with cudaHostRegister, so H2D/D2H DMA runs over
    2 MB pages (55 GB/s on the probe box; cudaHostAlloc'd buffers measured
    46-55 GB/s run to run, tools/upload_probe.py).  Falls back to torch's
    pinned allocator."""
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
            raise RuntimeError("cudaHostRegister failed")
        _HOST_KEEP.append(m)
        return t
    except Exception:
        return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
