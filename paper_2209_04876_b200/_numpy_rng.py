"""Bridge from NumPy's random API to the GPU's bit-exact PCG64 / ziggurat kernels.

The reference seeds every stream on the host through ``np.random.default_rng(seed)`` /
``SeedSequence.spawn`` (solvers.py:415-416, leverage.py:124, :217).  Seeding is host
orchestration: here it only turns a seed into PCG64's 128-bit (state, increment) pair, which
the CUDA kernels then advance and consume on the device (csrc/ks_rng.cu).

The ziggurat tables of ``Generator.standard_normal`` are data of the installed NumPy (2.3.5
in this image): they are read once from the local ``ki_double``/``wi_double``/``fi_double``
symbols of ``numpy/random/lib/libnpyrandom.a`` (an ar archive of ELF64 objects)."""

from __future__ import annotations

import struct
from functools import lru_cache
from pathlib import Path

import numpy as np

MASK64 = (1 << 64) - 1


_SS_STATES: dict = {}


def pcg64_state(seed):
    """(state, inc) of ``np.random.default_rng(seed)``'s PCG64 as Python ints."""
    if isinstance(seed, np.random.SeedSequence) and isinstance(seed.entropy, int):
        # pure function of the sequence's identity (entropy, spawn key, pool size): memoised
        key = (seed.entropy, tuple(seed.spawn_key), seed.pool_size, seed.n_children_spawned)
        got = _SS_STATES.get(key)
        if got is None:
            if len(_SS_STATES) > 1024:
                _SS_STATES.clear()
            st = np.random.PCG64(seed).state["state"]
            got = _SS_STATES[key] = (int(st["state"]), int(st["inc"]))
        return got
    if isinstance(seed, np.random.Generator):
        bg = seed.bit_generator
    elif isinstance(seed, np.random.BitGenerator):
        bg = seed
    else:
        bg = np.random.PCG64(seed)
    if not isinstance(bg, np.random.PCG64):
        raise TypeError(f"only PCG64 streams are supported on the device, got {type(bg).__name__}")
    st = bg.state["state"]
    return int(st["state"]), int(st["inc"])


def split128(x: int):
    return (x >> 64) & MASK64, x & MASK64


def _ar_members(blob: bytes):
    if not blob.startswith(b"!<arch>\n"):
        raise ValueError("not an ar archive")
    off = 8
    longnames = b""
    while off + 60 <= len(blob):
        hdr = blob[off:off + 60]
        name = hdr[:16].decode(errors="replace").strip()
        size = int(hdr[48:58].decode().strip())
        data = blob[off + 60: off + 60 + size]
        if name == "//":
            longnames = data
        elif name.startswith("/") and name[1:].isdigit() and longnames:
            start = int(name[1:])
            end = longnames.find(b"\n", start)
            name = longnames[start:end].decode().rstrip("/")
        yield name.rstrip("/"), data
        off += 60 + size + (size & 1)


def _elf_symbol_bytes(obj: bytes, wanted):
    if obj[:4] != b"\x7fELF" or obj[4] != 2 or obj[5] != 1:
        return {}
    e_shoff = struct.unpack_from("<Q", obj, 0x28)[0]
    e_shentsize, e_shnum, e_shstrndx = struct.unpack_from("<HHH", obj, 0x3A)
    shdrs = []
    for i in range(e_shnum):
        base = e_shoff + i * e_shentsize
        (sh_name, sh_type, sh_flags, sh_addr, sh_offset, sh_size, sh_link, sh_info,
         sh_addralign, sh_entsize) = struct.unpack_from("<IIQQQQIIQQ", obj, base)
        shdrs.append((sh_type, sh_offset, sh_size, sh_link, sh_entsize))
    out = {}
    for sh_type, sh_offset, sh_size, sh_link, sh_entsize in shdrs:
        if sh_type != 2:  # SHT_SYMTAB
            continue
        str_off = shdrs[sh_link][1]
        for k in range(sh_size // 24):
            st_name, st_info, st_other, st_shndx, st_value, st_size = struct.unpack_from(
                "<IBBHQQ", obj, sh_offset + 24 * k)
            end = obj.find(b"\0", str_off + st_name)
            name = obj[str_off + st_name:end].decode(errors="replace")
            if name in wanted and 0 < st_shndx < len(shdrs):
                sec_off = shdrs[st_shndx][1]
                out[name] = obj[sec_off + st_value: sec_off + st_value + st_size]
    return out


@lru_cache(maxsize=1)
def ziggurat_tables():
    """(ki uint64[256], wi float64[256], fi float64[256]) of the installed NumPy."""
    lib = Path(np.__file__).resolve().parent / "random" / "lib" / "libnpyrandom.a"
    blob = lib.read_bytes()
    wanted = {"ki_double", "wi_double", "fi_double"}
    found = {}
    for name, data in _ar_members(blob):
        if name.endswith(".o"):
            found.update(_elf_symbol_bytes(data, wanted))
        if wanted <= found.keys():
            break
    if not wanted <= found.keys():
        raise RuntimeError(f"ziggurat tables not found in {lib}")
    ki = np.frombuffer(found["ki_double"], dtype="<u8")[:256].copy()
    wi = np.frombuffer(found["wi_double"], dtype="<f8")[:256].copy()
    fi = np.frombuffer(found["fi_double"], dtype="<f8")[:256].copy()
    if ki.size != 256 or wi.size != 256 or fi.size != 256 or fi[0] != 1.0:
        raise RuntimeError("unexpected ziggurat table layout in libnpyrandom.a")
    return ki, wi, fi


_SS_INIT_A, _SS_MULT_A, _SS_INIT_B, _SS_MULT_B = 0x43b0d7e5, 0x931e8875, 0x8b51f9dd, 0x58f38ded
_SS_MIX_L, _SS_MIX_R = 0xca01f9dd, 0x4973f715


def seedseq_children_seed_words(entropy: int, count: int) -> np.ndarray:
    """PCG64 seeding words of ``np.random.SeedSequence(entropy).spawn(count)``, vectorised.

    Row i holds (initstate hi, initstate lo, initseq hi, initseq lo) = the four uint64 words of
    child i's ``generate_state(4, np.uint64)`` that ``PCG64(child)`` feeds to pcg64_set_seed; the
    device finishes the seeding (ks_pcg64_random_streams, seeded = 1).  Restates NumPy's
    published SeedSequence algorithm (entropy and spawn key as little-endian uint32 words, the
    run entropy zero-padded to the pool size, hashmix / mix over a 4-word pool, then the
    generate_state hash); checked bit for bit against NumPy in tests/test_rng_oracle.py."""
    if entropy < 0 or count >= 2 ** 32:
        raise ValueError("unsupported SeedSequence parameters")
    run = []
    e = int(entropy)
    while e > 0:
        run.append(e & 0xFFFFFFFF)
        e >>= 32
    run = run or [0]
    run += [0] * max(0, 4 - len(run))
    m32 = np.uint64(0xFFFFFFFF)
    sh16 = np.uint64(16)
    ent = np.zeros((count, len(run) + 1), dtype=np.uint64)
    ent[:, :len(run)] = np.asarray(run, dtype=np.uint64)
    ent[:, len(run)] = np.arange(count, dtype=np.uint64)
    hc = [_SS_INIT_A]

    def hashmix(v):
        v = (v ^ np.uint64(hc[0])) & m32
        hc[0] = (hc[0] * _SS_MULT_A) & 0xFFFFFFFF
        v = (v * np.uint64(hc[0])) & m32
        return v ^ (v >> sh16)

    def mix(x, y):
        r = (np.uint64(_SS_MIX_L) * x - np.uint64(_SS_MIX_R) * y) & m32
        return r ^ (r >> sh16)

    pool = [hashmix(ent[:, i]) for i in range(4)]
    for src in range(4):
        for dst in range(4):
            if src != dst:
                pool[dst] = mix(pool[dst], hashmix(pool[src]))
    for src in range(4, ent.shape[1]):
        for dst in range(4):
            pool[dst] = mix(pool[dst], hashmix(ent[:, src]))
    h = _SS_INIT_B
    w32 = []
    for i in range(8):
        v = pool[i % 4] ^ np.uint64(h)
        h = (h * _SS_MULT_B) & 0xFFFFFFFF
        v = (v * np.uint64(h)) & m32
        w32.append(v ^ (v >> sh16))
    out = np.empty((count, 4), dtype=np.uint64)
    for k in range(4):
        out[:, k] = (w32[2 * k + 1] << np.uint64(32)) | w32[2 * k]
    return out
