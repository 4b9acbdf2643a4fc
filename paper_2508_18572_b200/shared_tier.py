"""One host tier shared by several processes (R28): every tensor-parallel rank maps the
same file-backed region (e.g. under /dev/shm or a hugetlbfs mount) and registers it with its own
pool as caller-owned memory (``HostPool(host=..., host_heads=Ht, head_begin=h0)``), so a node keeps
ONE copy of the KV of all heads while each GPU pulls its head slice over its own link.

Plumbing only (file creation and mapping): no layout or address arithmetic lives here.
"""
from __future__ import annotations

import mmap
import os

import numpy as np


class SharedTier:
    """A MAP_SHARED mapping of ``path`` holding ``nbytes``; ``create`` sizes (and zero-fills) the
    file, the other ranks open it after a barrier.  ``.array`` is a uint8 numpy view to pass as
    ``HostPool(host=...)``; the creator unlinks the file in :meth:`close` (``unlink=True``)."""

    def __init__(self, path: str, nbytes: int, create: bool):
        self.path, self.nbytes, self.creator = path, int(nbytes), create
        flags = os.O_RDWR | (os.O_CREAT | os.O_TRUNC if create else 0)
        fd = os.open(path, flags, 0o600)
        try:
            if create:
                os.ftruncate(fd, self.nbytes)
            elif os.fstat(fd).st_size < self.nbytes:
                raise ValueError(f"{path}: {os.fstat(fd).st_size} bytes, need {self.nbytes}")
            self._mm = mmap.mmap(fd, self.nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        finally:
            os.close(fd)
        self.array = np.frombuffer(self._mm, dtype=np.uint8, count=self.nbytes)

    def close(self, unlink: bool = True) -> None:
        if self._mm is None:
            return
        self.array = None
        try:
            self._mm.close()
        except BufferError:   # a numpy view is still alive somewhere; the OS unmaps at exit
            pass
        self._mm = None
        if unlink and self.creator:
            try:
                os.unlink(self.path)
            except FileNotFoundError:
                pass


def free_bytes(directory: str) -> int:
    st = os.statvfs(directory)
    return st.f_bavail * st.f_frsize
