"""Analytic machine model (drop-in for mktune.hardware, hardware.py:35-111).

The nine integer fields and their validation are the reference's. The B200
re-parameterisation adds OPTIONAL tcgen05 fields (TMEM columns, MMA atom
shapes, TMA swizzle). A descriptor without them behaves exactly like the
reference ("parity mode"); with them, the planner additionally keeps only
uKernel tiles that map onto tcgen05 MMA tiles ("B200 mode",
``tcgen05_mode``), applied right after enumeration.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, fields
from pathlib import Path

from .errors import InputError

INT_FIELDS = (
    "num_cores",
    "regs_per_core",
    "smem_per_core_bytes",
    "global_bw_bytes_per_s",
    "shared_bw_bytes_per_s",
    "peak_flops",
    "default_active_blocks",
    "active_blocks_per_core",
    "align_elems",
)
# sm_100a extension fields and their sm_100a values (b200_bf16(tcgen05=True));
# other values re-parameterise the legality rules (planner.cpp tcgen05_legal)
# within what the executor can run (validated below)
EXT_FIELDS = {
    "tmem_columns": 512,
    "mma_m_atoms": (64, 128),
    "mma_n_step": 16,
    "mma_n_max": 256,
    "tma_swizzle_bytes": 128,
}


@dataclass(frozen=True)
class HardwareDescriptor:
    """Frozen machine model; safe to share between tuning threads."""

    name: str
    num_cores: int
    regs_per_core: int
    smem_per_core_bytes: int
    global_bw_bytes_per_s: int
    shared_bw_bytes_per_s: int
    peak_flops: int
    default_active_blocks: int
    active_blocks_per_core: int
    align_elems: int
    tmem_columns: int | None = None
    mma_m_atoms: tuple | None = None
    mma_n_step: int | None = None
    mma_n_max: int | None = None
    tma_swizzle_bytes: int | None = None

    def __post_init__(self):
        if not isinstance(self.name, str) or not self.name:
            raise InputError("descriptor field 'name' must be a non-empty string", field="name")
        for f in INT_FIELDS:
            v = getattr(self, f)
            if isinstance(v, bool) or not isinstance(v, int):
                raise InputError(f"descriptor field '{f}' must be an integer", field=f)
            if v <= 0:
                raise InputError(f"descriptor field '{f}' must be strictly positive, got {v}", field=f)
        if self.align_elems & (self.align_elems - 1):
            raise InputError(
                f"descriptor field 'align_elems' must be a power of two, got {self.align_elems}", field="align_elems"
            )
        if isinstance(self.mma_m_atoms, list):
            object.__setattr__(self, "mma_m_atoms", tuple(self.mma_m_atoms))
        set_ext = [k for k in EXT_FIELDS if getattr(self, k) is not None]
        if set_ext and len(set_ext) != len(EXT_FIELDS):
            missing = [k for k in EXT_FIELDS if getattr(self, k) is None][0]
            raise InputError(f"tcgen05 extension field '{missing}' is missing", field=missing)
        if set_ext:
            self._check_tcgen05()

    def _check_tcgen05(self) -> None:
        """The executor's limits on the tcgen05 fields (sm_100a kind::f16,
        cta_group::1): M atoms from {64, 128}; N step 8 or 16; widest N a
        multiple of the step up to 256; TMEM a power of two holding two
        widest accumulators, at most 512 columns; a 32/64/128-B swizzle."""
        atoms = self.mma_m_atoms
        if not isinstance(atoms, tuple) or not atoms or any(a not in (64, 128) for a in atoms):
            raise InputError("tcgen05 extension field 'mma_m_atoms' must be a non-empty subset of (64, 128)",
                             field="mma_m_atoms")
        step, nmax, cols, swz = self.mma_n_step, self.mma_n_max, self.tmem_columns, self.tma_swizzle_bytes
        for k, v in (("mma_n_step", step), ("mma_n_max", nmax), ("tmem_columns", cols), ("tma_swizzle_bytes", swz)):
            if isinstance(v, bool) or not isinstance(v, int) or v <= 0:
                raise InputError(f"tcgen05 extension field '{k}' must be a positive integer", field=k)
        if step not in (8, 16):
            raise InputError("tcgen05 extension field 'mma_n_step' must be 8 or 16", field="mma_n_step")
        if nmax % step or not 2 * step <= nmax <= 256:
            raise InputError("tcgen05 extension field 'mma_n_max' must be a multiple of mma_n_step in [2*step, 256]",
                             field="mma_n_max")
        if cols & (cols - 1) or not 2 * nmax <= cols <= 512:
            raise InputError("tcgen05 extension field 'tmem_columns' must be a power of two in [2*mma_n_max, 512]",
                             field="tmem_columns")
        if swz not in (32, 64, 128):
            raise InputError("tcgen05 extension field 'tma_swizzle_bytes' must be 32, 64 or 128",
                             field="tma_swizzle_bytes")

    @property
    def total_active_blocks(self) -> int:
        """One wave: cores x active blocks per core (hardware.py:63-66)."""
        return self.num_cores * self.active_blocks_per_core

    @property
    def tcgen05_mode(self) -> bool:
        return self.tmem_columns is not None

    def to_doc(self) -> dict:
        doc = {}
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name in EXT_FIELDS and v is None:
                continue
            doc[f.name] = list(v) if isinstance(v, tuple) else v
        return doc

    def parity(self) -> "HardwareDescriptor":
        """The same machine without the tcgen05 extension (reference semantics)."""
        return HardwareDescriptor(**{f: getattr(self, f) for f in ("name",) + INT_FIELDS})


def load_hardware_descriptor(document: str | bytes | dict) -> HardwareDescriptor:
    """Parse JSON text or a dict; unknown fields are rejected by name."""
    if isinstance(document, (str, bytes)):
        try:
            tree = json.loads(document)
        except json.JSONDecodeError as exc:
            raise InputError(f"malformed hardware descriptor document: {exc}") from exc
    else:
        tree = document
    if not isinstance(tree, dict):
        raise InputError("hardware descriptor document must be a JSON object")
    required = {"name", *INT_FIELDS}
    allowed = required | set(EXT_FIELDS)
    extra = sorted(set(tree) - allowed)
    if extra:
        raise InputError(f"unknown hardware descriptor field '{extra[0]}'", field=extra[0])
    absent = sorted(required - set(tree))
    if absent:
        raise InputError(f"missing hardware descriptor field '{absent[0]}'", field=absent[0])
    return HardwareDescriptor(**tree)


def load_hardware_file(path: str | Path) -> HardwareDescriptor:
    p = Path(path)
    if not p.exists():
        raise InputError(f"hardware descriptor file not found: {p}", field="hardware")
    return load_hardware_descriptor(p.read_text())


def canonical_document(tree: dict) -> str:
    """Sorted keys, two-space indent, trailing newline (hardware.py:109-111)."""
    return json.dumps(tree, sort_keys=True, indent=2) + "\n"


def serialize_hardware_descriptor(descriptor: HardwareDescriptor) -> str:
    return canonical_document(descriptor.to_doc())


# ---------------------------------------------------------------- sm_100a presets
# SURVEY.md Appendix A. peak_flops uses the MEASURED dense bf16 GEMM rate of
# this pool's B200s (MEASURED_PEAKS.json bf16_tflops = 1649.8 TF/s); the FFMA
# figure is 148 SMs x 128 FMA/clk x 2 x 1.965 GHz.

def b200_bf16(tcgen05: bool = True) -> HardwareDescriptor:
    ext = dict(EXT_FIELDS) if tcgen05 else {}
    return HardwareDescriptor(
        name="b200-sm100a-bf16" + ("" if tcgen05 else "-parity"),
        num_cores=148,
        regs_per_core=65536,
        smem_per_core_bytes=232448,
        global_bw_bytes_per_s=8_000_000_000_000,
        shared_bw_bytes_per_s=37_225_920_000_000,
        peak_flops=1_649_800_000_000_000,
        default_active_blocks=1,
        active_blocks_per_core=1,
        align_elems=64,
        **ext,
    )


def b200_ffma() -> HardwareDescriptor:
    return HardwareDescriptor(
        name="b200-sm100a-ffma",
        num_cores=148,
        regs_per_core=65536,
        smem_per_core_bytes=232448,
        global_bw_bytes_per_s=8_000_000_000_000,
        shared_bw_bytes_per_s=37_225_920_000_000,
        peak_flops=74_449_920_000_000,
        default_active_blocks=2,
        active_blocks_per_core=2,
        align_elems=32,
    )
