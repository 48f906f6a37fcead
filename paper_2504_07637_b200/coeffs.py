"""Coefficient dataset: bit-exact text persistence, kernel tables, header codegen.

Mirrors the SPEC ``coeffs`` module, which the reference
declares but does not ship:

* ``Dataset`` / ``Record``            -- SPEC.md:220-223 (one record per order n)
* ``save`` / ``load``                 -- SPEC.md:230-238 (versioned line-oriented text,
                                         lowercase hex-float literals, '#' comments,
                                         trailing whole-file checksum)
* ``build_kernel_table``              -- SPEC.md:239-247 (flat per-n arrays + counts)
* ``gen_header``                      -- SPEC.md:248-256 (generated source; here a C++
                                         header of ``__constant__`` tables and per-order
                                         factor counts consumed by the sm_100a kernels)

The file stores every real already rounded ONCE from the fit precision to the
profile's target precision, so loading is exact and the kernel
table is the identity on the stored values.  ``float.hex`` is the canonical
literal form (``1.0 -> 0x1.0000000000000p+0``), which C99/C++17 parse exactly.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass, field
from pathlib import Path

FORMAT_VERSION = 1
PROFILES = {"double53": 53, "single24": 24}
DATA_DIR = Path(__file__).resolve().parent / "data"


class DatasetError(ValueError):
    """Malformed, truncated, version- or checksum-mismatched dataset file."""


def to_f32(v: float) -> float:
    """Exact binary32 value (v must already be a binary32 number)."""
    r = struct.unpack("<f", struct.pack("<f", v))[0]
    if r != v:
        raise DatasetError(f"{v!r} is not representable in binary32")
    return r


@dataclass
class Record:
    """One fitted order: constants, cut-off, root-factored form (Eqs. 12-14)."""

    n: int
    N: int
    c: float            # c_n (Eq. 3)
    q0: float           # Q_n(0) (Eq. 9)
    q1: float           # Q'_n(0) (Eq. 10)
    q2: float           # alpha_n - q1
    alpha: float
    beta: float
    z: float            # cut-off z_{n,b} (Eq. 17, b = profile bits)
    x_up: float         # above this x the asymptotic branch recurs upward (underflow guard)
    u_quads: list = field(default_factory=list)   # [(y, a)] -> (x-y)^2 + a
    u_lins: list = field(default_factory=list)    # [y]      -> (x-y)
    v_quads: list = field(default_factory=list)   # [(z, b)]
    v_lins: list = field(default_factory=list)    # [z]
    exact_bits: float = 0.0                       # -log2 E_n of the fit (Eq. 15)

    def counts(self):
        return (len(self.u_quads), len(self.u_lins), len(self.v_quads), len(self.v_lins))

    def reals(self):
        out = [self.c, self.q0, self.q1, self.q2, self.alpha, self.beta, self.z, self.x_up]
        for y, a in self.u_quads:
            out += [y, a]
        out += list(self.u_lins)
        for y, a in self.v_quads:
            out += [y, a]
        out += list(self.v_lins)
        return out


@dataclass
class Dataset:
    profile: str
    records: dict = field(default_factory=dict)   # n -> Record
    version: int = FORMAT_VERSION

    @property
    def bits(self):
        return PROFILES[self.profile]

    def orders(self):
        return sorted(self.records)

    def __eq__(self, other):
        if not isinstance(other, Dataset):
            return NotImplemented
        if (self.profile, self.version, self.orders()) != (other.profile, other.version,
                                                           other.orders()):
            return False
        for n in self.orders():
            a, b = self.records[n], other.records[n]
            if a.N != b.N or a.counts() != b.counts():
                return False
            ra, rb = a.reals(), b.reals()
            if any(struct.pack("<d", x) != struct.pack("<d", y) for x, y in zip(ra, rb)):
                return False
        return True


def _hex(v: float) -> str:
    return float(v).hex()


def dumps(ds: Dataset) -> str:
    if ds.profile not in PROFILES:
        raise DatasetError(f"unknown profile {ds.profile!r}")
    lines = [
        "# Boys-function Q~_n approximation dataset (Laikov, arXiv 2504.07637, Eqs. 12-14)",
        "# reals are hex floats rounded once to the profile precision",
        f"version {ds.version}",
        f"profile {ds.profile}",
        f"orders {len(ds.records)}",
    ]
    for n in ds.orders():
        r = ds.records[n]
        if ds.profile == "single24":
            for v in r.reals():
                to_f32(v)
        lines.append(f"record {r.n} {r.N}")
        for name in ("c", "q0", "q1", "q2", "alpha", "beta", "z", "x_up"):
            lines.append(f"  {name} {_hex(getattr(r, name))}")
        lines.append(f"  exact_bits {r.exact_bits:.3f}")
        lines.append(f"  u_quads {len(r.u_quads)}")
        lines += [f"    {_hex(y)} {_hex(a)}" for y, a in r.u_quads]
        lines.append(f"  u_lins {len(r.u_lins)}")
        lines += [f"    {_hex(y)}" for y in r.u_lins]
        lines.append(f"  v_quads {len(r.v_quads)}")
        lines += [f"    {_hex(y)} {_hex(a)}" for y, a in r.v_quads]
        lines.append(f"  v_lins {len(r.v_lins)}")
        lines += [f"    {_hex(y)}" for y in r.v_lins]
        lines.append("end")
    body = "\n".join(lines) + "\n"
    digest = hashlib.sha256(body.encode()).hexdigest()
    return body + f"checksum sha256 {digest}\n"


def save(ds: Dataset, path) -> None:
    Path(path).write_text(dumps(ds))


def _parse_real(tok: str, lineno: int) -> float:
    try:
        if not tok.startswith(("0x", "-0x")):
            raise ValueError
        return float.fromhex(tok)
    except ValueError:
        raise DatasetError(f"line {lineno}: malformed hex-float literal {tok!r}") from None


def loads(text: str) -> Dataset:
    lines = text.split("\n")
    if not text.endswith("\n") or len(lines) < 2:
        raise DatasetError("truncated dataset (no trailing newline)")
    last = lines[-2]
    if not last.startswith("checksum sha256 "):
        raise DatasetError("truncated dataset (missing checksum line)")
    body = text[: len(text) - len(last) - 1]
    if hashlib.sha256(body.encode()).hexdigest() != last.split()[-1]:
        raise DatasetError("checksum mismatch")
    toks = []
    for i, ln in enumerate(lines[:-2], start=1):
        s = ln.split("#", 1)[0].strip()
        if s:
            toks.append((i, s.split()))
    pos = 0

    def take(key, nargs):
        nonlocal pos
        if pos >= len(toks):
            raise DatasetError(f"unexpected end of dataset, wanted {key!r}")
        ln, t = toks[pos]
        if key is not None and t[0] != key:
            raise DatasetError(f"line {ln}: expected {key!r}, got {t[0]!r}")
        if len(t) != nargs + (0 if key is None else 1):
            raise DatasetError(f"line {ln}: wrong field count")
        pos += 1
        return ln, (t if key is None else t[1:])

    ln, (ver,) = take("version", 1)
    if int(ver) != FORMAT_VERSION:
        raise DatasetError(f"line {ln}: version {ver} != supported {FORMAT_VERSION}")
    ln, (prof,) = take("profile", 1)
    if prof not in PROFILES:
        raise DatasetError(f"line {ln}: unknown profile {prof!r}")
    _, (cnt,) = take("orders", 1)
    ds = Dataset(profile=prof, version=int(ver))
    for _ in range(int(cnt)):
        ln, (n, N) = take("record", 2)
        vals = {}
        for name in ("c", "q0", "q1", "q2", "alpha", "beta", "z", "x_up"):
            ln, (v,) = take(name, 1)
            vals[name] = _parse_real(v, ln)
        _, (eb,) = take("exact_bits", 1)
        groups = {}
        for name, width in (("u_quads", 2), ("u_lins", 1), ("v_quads", 2), ("v_lins", 1)):
            _, (k,) = take(name, 1)
            items = []
            for _ in range(int(k)):
                ln, t = take(None, width)
                vs = [_parse_real(x, ln) for x in t]
                items.append(tuple(vs) if width == 2 else vs[0])
            groups[name] = items
        take("end", 0)
        rec = Record(n=int(n), N=int(N), exact_bits=float(eb), **vals, **groups)
        if prof == "single24":
            for v in rec.reals():
                to_f32(v)
        if rec.n in ds.records:
            raise DatasetError(f"duplicate record for n={rec.n}")
        ds.records[rec.n] = rec
    if pos != len(toks):
        raise DatasetError(f"line {toks[pos][0]}: trailing content")
    return ds


def load(path) -> Dataset:
    return loads(Path(path).read_text())


def default_path(profile: str) -> Path:
    return DATA_DIR / f"boys_{profile}.dat"


def load_default(profile: str) -> Dataset:
    return load(default_path(profile))


# ----------------------------------------------------------------------------
# KernelTable and generated source
# ----------------------------------------------------------------------------

MAX_QUADS = 8      # per polynomial; N <= 16 gives at most 8 quadratic factors
MAX_LINS = 2


@dataclass
class KernelTable:
    """Flat per-n arrays + counts for one profile."""

    profile: str
    orders: list
    counts: list        # [(L_u, l_u, L_v, l_v)] per order
    rows: list          # per order: dict of scalars and padded factor arrays

    @property
    def max_order(self):
        return self.orders[-1]


def build_kernel_table(ds: Dataset) -> KernelTable:
    orders = ds.orders()
    if orders != list(range(len(orders))):
        raise DatasetError("kernel table needs contiguous orders 0..n_max")
    rows, counts = [], []
    for n in orders:
        r = ds.records[n]
        Lu, lu, Lv, lv = r.counts()
        if 2 * Lu + lu != r.N - 1 or 2 * Lv + lv != r.N:
            raise DatasetError(f"n={n}: factor degrees do not match N={r.N}")
        if max(Lu, Lv) > MAX_QUADS or max(lu, lv) > MAX_LINS:
            raise DatasetError(f"n={n}: too many factors for the kernel layout")
        pad = lambda xs, k, w: list(xs) + [((0.0, 0.0) if w == 2 else 0.0)] * (k - len(xs))
        rows.append(dict(q0=r.q0, q1=r.q1, q2=r.q2, c=r.c, z=r.z, x_up=r.x_up,
                         uq=pad(r.u_quads, MAX_QUADS, 2), ul=pad(r.u_lins, MAX_LINS, 1),
                         vq=pad(r.v_quads, MAX_QUADS, 2), vl=pad(r.v_lins, MAX_LINS, 1)))
        counts.append((Lu, lu, Lv, lv))
    return KernelTable(profile=ds.profile, orders=orders, counts=counts, rows=rows)


def pack_rows(kt: KernelTable) -> bytes:
    """The table as the kernels hold it: one ``BoysRow<T>`` per order
    (csrc/boys_eval.cuh field order -- q0 q1 q2 c z x_up, uq[8][2], ul[2],
    vq[8][2], vl[2] in T, then cnt[4] int32; no padding for either T).
    Uploaded verbatim by ``boys_table_create``; its SHA-256 identifies a table."""
    fmt = "<42f4i" if kt.profile == "single24" else "<42d4i"
    out = []
    for row, cnt in zip(kt.rows, kt.counts):
        vals = [row[k] for k in ("q0", "q1", "q2", "c", "z", "x_up")]
        vals += [v for pair in row["uq"] for v in pair] + list(row["ul"])
        vals += [v for pair in row["vq"] for v in pair] + list(row["vl"])
        out.append(struct.pack(fmt, *vals, *cnt))
    return b"".join(out)


def table_checksum(kt: KernelTable) -> str:
    """SHA-256 of ``pack_rows(kt)`` (libboys exports the compiled table's
    digest as ``boys_table_checksum``)."""
    return hashlib.sha256(pack_rows(kt)).hexdigest()


def _lit(v: float, single: bool) -> str:
    s = float(v).hex()
    return s + ("f" if single else "")


def gen_header(tables: list) -> str:
    """C++ header with __constant__ rows and constexpr factor counts.

    One ``BoysRow<T>`` per order, field order fixed (see csrc/boys_eval.cuh).
    """
    out = ["// GENERATED by paper_2504_07637_b200.coeffs.gen_header -- do not edit.",
           "// Source: paper_2504_07637_b200/data/boys_*.dat (hex floats, rounded once).",
           "#pragma once",
           f"#define BOYS_MAX_QUADS {MAX_QUADS}",
           f"#define BOYS_MAX_LINS {MAX_LINS}",
           ""]
    for kt in tables:
        single = kt.profile == "single24"
        T = "float" if single else "double"
        tag = "F32" if single else "F64"
        nmax = kt.max_order
        out.append(f"#define BOYS_{tag}_MAX_ORDER {nmax}")
        out.append(f'#define BOYS_{tag}_TABLE_SHA256 "{table_checksum(kt)}"')
        out.append(f"// counts per order: {{u quads, u lins, v quads, v lins}}")
        out.append(f"__host__ __device__ constexpr int boys_shape_{tag.lower()}(int n, int k) {{")
        out.append(f"  constexpr int s[{nmax + 1}][4] = {{")
        out += [f"    {{{a}, {b}, {c}, {d}}},  // n={n}" for n, (a, b, c, d) in
                zip(kt.orders, kt.counts)]
        out.append("  };")
        out.append("  return s[n][k];")
        out.append("}")
        out.append(f"__constant__ BoysRow<{T}> kBoysRow{tag}[{nmax + 1}] = {{")
        for n, row in zip(kt.orders, kt.rows):
            sc = ", ".join(_lit(row[k], single) for k in ("q0", "q1", "q2", "c", "z", "x_up"))
            uq = ", ".join(f"{{{_lit(y, single)}, {_lit(a, single)}}}" for y, a in row["uq"])
            vq = ", ".join(f"{{{_lit(y, single)}, {_lit(a, single)}}}" for y, a in row["vq"])
            ul = ", ".join(_lit(y, single) for y in row["ul"])
            vl = ", ".join(_lit(y, single) for y in row["vl"])
            cn = ", ".join(str(k) for k in kt.counts[kt.orders.index(n)])
            out.append(f"  {{ /* n={n} */ {sc},\n    {{{uq}}},\n    {{{ul}}},\n"
                       f"    {{{vq}}},\n    {{{vl}}},\n    {{{cn}}} }},")
        out.append("};")
        out.append("")
    return "\n".join(out)
