"""Generate straight-line, structure-folded per-robot dynamics routines.

Why: the template kernels (vd_algos.cuh) carry per-value "may be non-zero"
flags through arrays; for a 29-joint tree those arrays stay in local memory,
the flags become runtime values and the compiled ABA is ~30 K SASS
instructions of which only ~4.6 K are FP64 (the rest select/flag traffic).
Here the recursion is unrolled in Python over a symbolic scalar instead:
every product with a structural 0 / ±1 of the model (axis-aligned joints,
identity offset rotations, zero offsets, sparse and massless inertias) is
folded at generation time, and the emitted C++ is plain SSA arithmetic on T.

The math mirrors vd_device.cuh / vd_algos.cuh term by term (same spatial
algebra, same transform stages X = X_off ∘ X_J, kinematics.hpp:35-38), so the
generated routine computes what `aba_one` computes:

  ABA (Featherstone RBDA Table 7.1; oracle: forward_dynamics,
  dynamics.hpp:421-444).  Pass 1 and pass 2 are fused as a DFS: a joint's
  velocity is computed on the way down and consumed by its pass-2 step on the
  way up, so only the velocities on the current root->leaf path are live.
  Pass-2 -> pass-3 state per joint (U/D, u/D and the joint's cos/sin or q) is
  written through `cx.st(k, v)` / read back with `cx.get(k)`: the kernel
  decides where slot k lives (registers, shared memory or an L2-resident
  scratch), because for a 29-joint tree it does not fit in registers.

Model constants come from the library's own packer (`packed_model`,
vdi_model_packed), so the generated code is the packed device model frozen
into code.  tools/gen_tree_kernels.py writes the builtin robots' routines
(vd_gen_robots.cuh); paper_2604_04310_b200/jit.py the routines of any other
model at load time.
"""
import ctypes
import os

SNAP = 1e-15


def _snap(x):
    for t in (0.0, 1.0, -1.0):
        if abs(x - t) < SNAP:
            return t
    return x


def packed_model(lib, h):
    """The packed device model of a host model handle (vdi_model_packed, the
    packer vd_device_model_create uses) as the generator's dict.  Values within
    1e-15 of 0 / ±1 are snapped (cos(π/2) residues) so their terms fold."""
    M = 64
    n = ctypes.c_int()
    par = (ctypes.c_int * M)()
    kind = (ctypes.c_int * M)()
    code = (ctypes.c_int * M)()
    axis = (ctypes.c_double * (3 * M))()
    R = (ctypes.c_double * (9 * M))()
    p = (ctypes.c_double * (3 * M))()
    inertia = (ctypes.c_double * (10 * M))()
    if lib.vdi_model_packed(h, ctypes.byref(n), par, kind, code, axis, R, p, inertia) != 0:
        raise RuntimeError(lib.vd_last_error().decode())
    n = n.value
    return dict(n=n, parent=list(par[:n]), kind=list(kind[:n]), code=list(code[:n]),
                axis=[_snap(v) for v in axis[:3 * n]], R=[_snap(v) for v in R[:9 * n]],
                p=[_snap(v) for v in p[:3 * n]], inertia=[_snap(v) for v in inertia[:10 * n]],
                fp=lib.vdi_model_fingerprint(h))


class Ex:
    """Symbolic scalar: a compile-time constant (c) or a named SSA value (s)."""

    __slots__ = ("c", "s")

    def __init__(self, c=None, s=None):
        self.c = c
        self.s = s

    def is0(self):
        return self.c is not None and self.c == 0.0


def K(x):
    return Ex(c=float(x))


ZERO = K(0.0)
ONE = K(1.0)


# Model constants shared by every routine of the robot being generated.  An
# fp64 literal costs up to two UMOVs per use in SASS (12 % of the G1 ABA's
# instructions); a __constant__ table read in C++ is hoisted out of the
# persistent loop into registers and spilled (round 1: tree29 RNEA 0.14 ->
# 0.20 ms).  VD_GEN_POOL=asm emits one opaque `ld.const` per use instead
# (LDCU.128 into uniform registers, two constants per instruction); round 2,
# tools/async_sweep.cu: G1 ABA 0.294 -> 0.290 ms, G1 RNEA 0.099 -> 0.116,
# Panda ABA 0.539 -> 0.571, G1 OSC 0.61 -> 0.67 ms.  Literals stay the default.
#
# Per routine (POOL_OPS, round 2): the G1 ABA reads its constants from the
# robot's __constant__ table with plain C++ reads and runs through k_gen_call,
# which calls the routine once per state out of line, so there is no loop to
# hoist the table reads out of and ptxas folds them into the DFMAs as
# constant-bank operands (tools/call_sweep.cu: 0.261 -> 0.242 ms fp64; the
# Panda ABA, the G1 RNEA / CRBA / FK and the fp32 routines measured no gain or
# a loss with it).
POOL = {}
POOL_MODE = os.environ.get("VD_GEN_POOL", "")  # "" literals, "asm" opaque ld.const, "table" plain table reads
USE_POOL = POOL_MODE in ("asm", "table")
POOL_OPS = {"tree29": ("Aba", "AbaFext")}
if os.environ.get("VD_GEN_POOL_OPS") is not None:  # experiments: "robot:Op,Op;robot:Op" ("Osc" = every OSC routine)
    POOL_OPS = {r: tuple(o.split(",")) for r, o in
                (e.split(":") for e in os.environ["VD_GEN_POOL_OPS"].split(";") if e)}
_POOL_ON = False  # set by emit_body while it generates a POOL_OPS routine


def _low32_zero(c):
    import struct
    return struct.unpack("<Q", struct.pack("<d", c))[0] & 0xFFFFFFFF == 0


class Gen:
    def __init__(self):
        self.lines = []
        self.n = 0
        self.flops = 0
        # scalar type of emitted temporaries: "T" (the kernel's dtype) or "TD"
        # (double) for the high-precision joints of a mixed-precision routine
        self.ty = "T"
        self.groups_read = set()  # input groups read through cx.x (see Algo.release)
        self.on_input = None  # Algo's read-after-release guard

    # ---------------------------------------------------------------- emission
    def lit(self, c):
        t = self.ty
        if c == 0.0:
            return f"{t}(0)"
        if c == 1.0:
            return f"{t}(1)"
        if c == -1.0:
            return f"{t}(-1)"
        if _low32_zero(c) or not (USE_POOL or _POOL_ON) or t != "T":  # immediate / literal
            return f"{t}({float.hex(c)})"
        if c not in POOL:
            POOL[c] = len(POOL)
        return f"kc<T, {POOL[c]}>()"

    def o(self, a):
        return a.s if a.c is None else self.lit(a.c)

    def tmp(self, expr, prefix="t", ty=None):
        name = f"{prefix}{self.n}"
        self.n += 1
        self.lines.append(f"  const {ty or self.ty} {name} = {expr};")
        return Ex(s=name)

    def raw(self, line):
        self.lines.append("  " + line)

    # ---------------------------------------------------------------- hooks (overridden by DGen for JVPs)
    def input(self, gi, i):
        self.groups_read.add(gi)
        if self.on_input:
            self.on_input(gi)
        return self.tmp(f"cx.x({gi}, {i})", "x", ty="T")

    def sincos(self, q, i):
        """(cos q, sin q) of joint i's angle, in the current precision."""
        self.raw(f"{self.ty} s{i}, c{i};")
        self.raw(f"vd_sincos_cx<Cx>({self.ty}({q.s}), &s{i}, &c{i});")
        return Ex(s=f"c{i}"), Ex(s=f"s{i}")

    def recip(self, d, prefix="di"):
        return self.tmp(f"{self.ty}(1) / {self.o(d)}", prefix)

    def sqrt(self, x):
        return self.tmp(f"vd_sqrt({self.o(x)})", "sq")

    def check_pos(self, d):
        self.raw(f"ok = ok && ({self.o(d)} > {self.ty}(0));")

    def check_finite(self, v):
        self.raw(f"ok = ok && vd_isfinite({self.o(v)});")

    def output(self, o, k, v):
        self.raw(f"cx.y({o}, {k}, {self.o(v)});")

    # ---------------------------------------------------------------- scalar ops (folding)
    def add(self, a, b):
        if a.c is not None and b.c is not None:
            return K(a.c + b.c)
        if a.is0():
            return b
        if b.is0():
            return a
        self.flops += 1
        return self.tmp(f"{self.o(a)} + {self.o(b)}")

    def sub(self, a, b):
        if a.c is not None and b.c is not None:
            return K(a.c - b.c)
        if b.is0():
            return a
        if a.is0():
            return self.neg(b)
        self.flops += 1
        return self.tmp(f"{self.o(a)} - {self.o(b)}")

    def neg(self, a):
        if a.c is not None:
            return K(-a.c)
        return self.tmp(f"-{a.s}")

    def mul(self, a, b):
        if a.c is not None and b.c is not None:
            return K(a.c * b.c)
        if a.is0() or b.is0():
            return ZERO
        if a.c == 1.0:
            return b
        if b.c == 1.0:
            return a
        if a.c == -1.0:
            return self.neg(b)
        if b.c == -1.0:
            return self.neg(a)
        self.flops += 1
        return self.tmp(f"{self.o(a)} * {self.o(b)}")

    def sum(self, xs):
        acc = ZERO
        for x in xs:
            acc = self.add(acc, x)
        return acc

    def dot(self, xs, ys):
        return self.sum([self.mul(x, y) for x, y in zip(xs, ys)])

    # ---------------------------------------------------------------- 3-vectors / 3x3 (row-major)
    def cross3(self, x, y):
        return [self.sub(self.mul(x[1], y[2]), self.mul(x[2], y[1])),
                self.sub(self.mul(x[2], y[0]), self.mul(x[0], y[2])),
                self.sub(self.mul(x[0], y[1]), self.mul(x[1], y[0]))]

    def matvec(self, Q, x):
        return [self.dot(Q[3 * r:3 * r + 3], x) for r in range(3)]

    def matTvec(self, Q, x):
        return [self.dot([Q[r], Q[3 + r], Q[6 + r]], x) for r in range(3)]

    def vadd(self, x, y):
        return [self.add(a, b) for a, b in zip(x, y)]

    def vsub(self, x, y):
        return [self.sub(a, b) for a, b in zip(x, y)]

    # ---------------------------------------------------------------- spatial (angular first: [a0 a1 a2 l0 l1 l2])
    def motion_in(self, Q, t, m):  # inverse_transform_motion (spatial.hpp:233-238)
        a = self.matTvec(Q, m[:3])
        d = self.vsub(m[3:], self.cross3(t, m[:3]))
        return a + self.matTvec(Q, d)

    def motion_out(self, Q, t, m):  # transform_motion (spatial.hpp:225-230)
        a = self.matvec(Q, m[:3])
        l = self.vadd(self.matvec(Q, m[3:]), self.cross3(t, a))
        return a + l

    def force_out(self, Q, t, f):  # transform_force (spatial.hpp:241-246)
        l = self.matvec(Q, f[3:])
        a = self.vadd(self.matvec(Q, f[:3]), self.cross3(t, l))
        return a + l

    def crm(self, v, m):  # spatial.hpp:204-208
        a = self.cross3(v[:3], m[:3])
        l = self.vadd(self.cross3(v[:3], m[3:]), self.cross3(v[3:], m[:3]))
        return a + l

    def crf(self, v, f):  # spatial.hpp:212-216
        a = self.vadd(self.cross3(v[:3], f[:3]), self.cross3(v[3:], f[3:]))
        l = self.cross3(v[:3], f[3:])
        return a + l

    def sdot(self, f, m):
        return self.add(self.dot(f[:3], m[:3]), self.dot(f[3:], m[3:]))

    # rigid-body inertia, 10 params: m, h[3], I = xx yy zz xy xz yz (about the origin)
    def rb_apply(self, b, v):
        m, h, I = b
        hv = self.cross3(h, v[3:])
        hw = self.cross3(h, v[:3])
        Im = [[I[0], I[3], I[4]], [I[3], I[1], I[5]], [I[4], I[5], I[2]]]
        a = [self.add(self.dot(Im[r], v[:3]), hv[r]) for r in range(3)]
        l = [self.sub(self.mul(m, v[3 + k]), hw[k]) for k in range(3)]
        return a + l

    # articulated inertia: dict A (sym 6: xx yy zz xy xz yz), B (3x3 row-major), C (sym 6)
    @staticmethod
    def sym(s6, r, c):
        return s6[r] if r == c else s6[r + c + 2]

    def ai_from_rb(self, b):
        m, h, I = b
        B = [ZERO, self.neg(h[2]), h[1], h[2], ZERO, self.neg(h[0]), self.neg(h[1]), h[0], ZERO]
        return {"A": list(I), "B": B, "C": [m, m, m, ZERO, ZERO, ZERO]}

    def ai_add(self, x, y):
        return {k: [self.add(a, b) for a, b in zip(x[k], y[k])] for k in ("A", "B", "C")}

    def ai_apply(self, I, v):
        A, B, C = I["A"], I["B"], I["C"]
        a = [self.add(self.dot([self.sym(A, r, 0), self.sym(A, r, 1), self.sym(A, r, 2)], v[:3]),
                      self.dot(B[3 * r:3 * r + 3], v[3:])) for r in range(3)]
        l = [self.add(self.dot([B[r], B[3 + r], B[6 + r]], v[:3]),
                      self.dot([self.sym(C, r, 0), self.sym(C, r, 1), self.sym(C, r, 2)], v[3:])) for r in range(3)]
        return a + l

    def sym_rotate(self, Q, s6):  # Q S Qᵀ
        s = [[self.sym(s6, r, c) for c in range(3)] for r in range(3)]
        t = [[self.dot(Q[3 * r:3 * r + 3], [s[0][c], s[1][c], s[2][c]]) for c in range(3)] for r in range(3)]
        ir, ic = (0, 1, 2, 0, 0, 1), (0, 1, 2, 1, 2, 2)
        return [self.dot(t[ir[k]], Q[3 * ic[k]:3 * ic[k] + 3]) for k in range(6)]

    def full_rotate(self, Q, B):  # Q B Qᵀ
        t = [[self.dot(Q[3 * r:3 * r + 3], [B[c], B[3 + c], B[6 + c]]) for c in range(3)] for r in range(3)]
        return [self.dot(t[r], Q[3 * c:3 * c + 3]) for r in range(3) for c in range(3)]

    def ai_out(self, I, Q, t):
        """X* IA X*ᵀ for X = (Q, t) (vd_device.cuh ai_out)."""
        o = {"A": self.sym_rotate(Q, I["A"]), "C": self.sym_rotate(Q, I["C"]), "B": self.full_rotate(Q, I["B"])}
        if all(x.is0() for x in t):
            return o
        C1 = [[self.sym(o["C"], r, c) for c in range(3)] for r in range(3)]
        B1 = o["B"]
        PC = [[None] * 3 for _ in range(3)]
        W = [[None] * 3 for _ in range(3)]
        Z = [[None] * 3 for _ in range(3)]
        for c in range(3):
            PC[0][c] = self.sub(self.mul(t[1], C1[2][c]), self.mul(t[2], C1[1][c]))
            PC[1][c] = self.sub(self.mul(t[2], C1[0][c]), self.mul(t[0], C1[2][c]))
            PC[2][c] = self.sub(self.mul(t[0], C1[1][c]), self.mul(t[1], C1[0][c]))
        for c in range(3):
            W[0][c] = self.sub(self.mul(t[1], B1[c * 3 + 2]), self.mul(t[2], B1[c * 3 + 1]))
            W[1][c] = self.sub(self.mul(t[2], B1[c * 3 + 0]), self.mul(t[0], B1[c * 3 + 2]))
            W[2][c] = self.sub(self.mul(t[0], B1[c * 3 + 1]), self.mul(t[1], B1[c * 3 + 0]))
        for r in range(3):
            Z[r][0] = self.sub(self.mul(PC[r][1], t[2]), self.mul(PC[r][2], t[1]))
            Z[r][1] = self.sub(self.mul(PC[r][2], t[0]), self.mul(PC[r][0], t[2]))
            Z[r][2] = self.sub(self.mul(PC[r][0], t[1]), self.mul(PC[r][1], t[0]))
        ir, ic = (0, 1, 2, 0, 0, 1), (0, 1, 2, 1, 2, 2)
        A = [self.add(o["A"][k], self.sub(self.add(W[ir[k]][ic[k]], W[ic[k]][ir[k]]), Z[ir[k]][ic[k]])) for k in range(6)]
        B = [self.add(B1[3 * r + c], PC[r][c]) for r in range(3) for c in range(3)]
        return {"A": A, "B": B, "C": o["C"]}


class DualEx:
    """Forward-mode dual scalar (dual.hpp:14-42): value and tangent, each a
    symbolic Ex (structural zeros fold in both)."""

    __slots__ = ("v", "t")

    def __init__(self, v, t):
        self.v = v
        self.t = t

    @property
    def c(self):  # a constant only when the tangent is exactly zero
        return self.v.c if (self.v.c is not None and self.t.is0()) else None

    @property
    def s(self):
        return None

    def is0(self):
        return self.v.is0() and self.t.is0()


def _lift(x):
    return x if isinstance(x, DualEx) else DualEx(x, ZERO)


class DGen(Gen):
    """Gen over dual numbers: every spatial-algebra routine of Gen runs
    unchanged (it is written with add / sub / mul / neg); the hooks load
    tangents (cx.dx), differentiate sin/cos and 1/x, and write the tangent
    outputs to output group 1 (the JVP of the same routine)."""

    def add(self, a, b):
        a, b = _lift(a), _lift(b)
        return DualEx(Gen.add(self, a.v, b.v), Gen.add(self, a.t, b.t))

    def sub(self, a, b):
        a, b = _lift(a), _lift(b)
        return DualEx(Gen.sub(self, a.v, b.v), Gen.sub(self, a.t, b.t))

    def neg(self, a):
        a = _lift(a)
        return DualEx(Gen.neg(self, a.v), Gen.neg(self, a.t))

    def mul(self, a, b):
        a, b = _lift(a), _lift(b)
        v = Gen.mul(self, a.v, b.v)
        t = Gen.add(self, Gen.mul(self, a.v, b.t), Gen.mul(self, a.t, b.v))
        return DualEx(v, t)

    def o(self, a):
        return Gen.o(self, a.v if isinstance(a, DualEx) else a)

    def input(self, gi, i):
        self.groups_read.add(gi)
        if self.on_input:
            self.on_input(gi)
        return DualEx(self.tmp(f"cx.x({gi}, {i})", "x", ty="T"), self.tmp(f"cx.dx({gi}, {i})", "dx", ty="T"))

    def sincos(self, q, i):
        c, sn = Gen.sincos(self, q.v, i)
        # d sin = cos dq, d cos = −sin dq (dual.hpp:97-102)
        return DualEx(c, Gen.neg(self, Gen.mul(self, sn, q.t))), DualEx(sn, Gen.mul(self, c, q.t))

    def recip(self, d, prefix="di"):
        r = Gen.recip(self, d.v, prefix)
        return DualEx(r, Gen.neg(self, Gen.mul(self, d.t, Gen.mul(self, r, r))))

    def sqrt(self, x):
        # d √x = dx / (2 √x) (dual.hpp sqrt)
        x = _lift(x)
        v = Gen.sqrt(self, x.v)
        return DualEx(v, Gen.mul(self, x.t, self.tmp(f"T(0.5) / {v.s}", "hs")))

    def check_pos(self, d):
        Gen.check_pos(self, d.v)

    def check_finite(self, v):
        Gen.check_finite(self, v.v)
        Gen.check_finite(self, v.t)

    def output(self, o, k, v):
        v = _lift(v)
        Gen.output(self, 0, k, v.v)
        Gen.output(self, 1, k, v.t)


def frame_joints(lib, h):
    """Joints carrying a named frame with a non-identity offset (fixed-joint
    fused frames such as `l_palm`, `head`), from the library's own model."""
    out = set()
    for k in range(lib.vd_model_frame_count(h)):
        buf = ctypes.create_string_buffer(256)
        j = ctypes.c_int()
        off = (ctypes.c_double * 12)()
        lib.vd_model_frame(h, k, buf, 256, ctypes.byref(j), off)
        ident = [1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0]
        if j.value >= 0 and any(abs(off[t] - ident[t]) > 0 for t in range(12)):
            out.add(j.value)
    return sorted(out)


class Robot:
    def __init__(self, d, fjoints=()):
        self.d = d
        self.frame_joints = list(fjoints)
        self.n = d["n"]
        self.parent = d["parent"]
        self.kind = d["kind"]
        self.children = [[] for _ in range(self.n)]
        self.roots = []
        for i, p in enumerate(self.parent):
            (self.children[p] if p >= 0 else self.roots).append(i)

    def lower_pattern(self):
        """Branch-sparse lower triangle of M in compressed-column order: (r, c)
        for c ascending, r ascending, c an ancestor of r or r itself.  Every
        other entry of M is an exact zero (dynamics.hpp:330-335,
        test_dynamics.cpp:200-216).  Same order as vd_model_crba_pattern."""
        out = []
        for c in range(self.n):
            for r in range(c, self.n):
                j = r
                while j >= 0 and j != c:
                    j = self.parent[j]
                if j == c:
                    out.append((r, c))
        return out

    def axis(self, i):
        return [K(v) for v in self.d["axis"][3 * i:3 * i + 3]]

    def QO(self, i):
        return [K(v) for v in self.d["R"][9 * i:9 * i + 9]]

    def tO(self, i):
        return [K(v) for v in self.d["p"][3 * i:3 * i + 3]]

    def rb(self, i):
        I = self.d["inertia"][10 * i:10 * i + 10]
        return (K(I[0]), [K(v) for v in I[1:4]], [K(v) for v in I[4:10]])


class Joint:
    """X_i = X_off ∘ X_J(q) for one joint, built from its motion values
    (c, s) (revolute) or q (prismatic)."""

    def __init__(self, g, rb, i, cs=None, q=None):
        self.g = g
        self.i = i
        self.prismatic = rb.kind[i] == 1
        ax = rb.axis(i)
        self.ax = ax
        self.QO, self.tO = rb.QO(i), rb.tO(i)
        if self.prismatic:
            self.QJ = [ONE if k % 4 == 0 else ZERO for k in range(9)]
            self.tJ = [g.mul(a, q) for a in ax]
        else:
            c, s = cs
            self.tJ = [ZERO, ZERO, ZERO]
            unit = [k for k in range(3) if not ax[k].is0()]
            if len(unit) == 1 and abs(ax[unit[0]].c) == 1.0:
                k = unit[0]
                k1, k2 = (k + 1) % 3, (k + 2) % 3
                sg = s if ax[k].c > 0 else g.neg(s)
                Q = [ZERO] * 9
                Q[k * 3 + k] = ONE
                Q[k1 * 3 + k1] = c
                Q[k2 * 3 + k2] = c
                Q[k1 * 3 + k2] = g.neg(sg)
                Q[k2 * 3 + k1] = sg
                self.QJ = Q
            else:  # Rodrigues (spatial.hpp:302-308)
                omc = g.sub(ONE, c)
                Q = [g.add(g.mul(g.mul(ax[r], ax[cc]), omc), c if r == cc else ZERO) for r in range(3) for cc in range(3)]
                Q[1] = g.sub(Q[1], g.mul(ax[2], s))
                Q[2] = g.add(Q[2], g.mul(ax[1], s))
                Q[3] = g.add(Q[3], g.mul(ax[2], s))
                Q[5] = g.sub(Q[5], g.mul(ax[0], s))
                Q[6] = g.sub(Q[6], g.mul(ax[1], s))
                Q[7] = g.add(Q[7], g.mul(ax[0], s))
                self.QJ = Q

    def motion_to_child(self, m):
        g = self.g
        return g.motion_in(self.QJ, self.tJ, g.motion_in(self.QO, self.tO, m))

    def motion_to_parent(self, m):
        g = self.g
        return g.motion_out(self.QO, self.tO, g.motion_out(self.QJ, self.tJ, m))

    def force_to_parent(self, f):
        g = self.g
        return g.force_out(self.QO, self.tO, g.force_out(self.QJ, self.tJ, f))

    def ai_to_parent(self, I):
        g = self.g
        return g.ai_out(g.ai_out(I, self.QJ, self.tJ), self.QO, self.tO)

    # motion subspace S: (axis, 0) revolute / (0, axis) prismatic
    def S(self, x):
        m = [self.g.mul(a, x) for a in self.ax]
        return ([ZERO] * 3 + m) if self.prismatic else (m + [ZERO] * 3)

    def Svec(self):
        return ([ZERO] * 3 + self.ax) if self.prismatic else (self.ax + [ZERO] * 3)

    def Sdot(self, f):
        return self.g.dot(self.ax, f[3:] if self.prismatic else f[:3])


class Algo:
    """Shared emission state of one generated routine: the symbolic
    generator, slot allocation (cx.st / cx.get) and the prologue that parks
    every joint's motion values (cos/sin, or q for prismatic joints) and,
    optionally, q̇ in the first slots."""

    def __init__(self, rb, with_qd_slots, hp=(), extra=(), dual=False, only=None):
        """extra: further input groups (2 = q̈ or τ) loaded by the prologue
        into slots (self.xrefs[(g, i)]); dual: emit the forward-mode JVP."""
        self.rb = rb
        self.g = DGen() if dual else Gen()
        self.nslot = 0
        self.hp = set(hp)  # joints computed in double when T is float
        self.mrefs, self.qdrefs, self.xrefs = {}, {}, {}
        g = self.g
        g.raw("using TD = double;")
        g.raw("bool ok = true;")
        # every input load of the state is issued first (all in flight at
        # once), then n independent sincos chains
        joints = [i for i in range(rb.n) if only is None or i in only]  # prologue subset
        qv = {i: g.input(0, i) for i in joints}
        qdv = {i: g.input(1, i) for i in joints} if with_qd_slots else {}
        xv = {(gi, i): g.input(gi, i) for gi in extra for i in joints}
        for i in joints:
            g.ty = "TD" if i in self.hp else "T"
            qi = qv[i]
            if rb.kind[i] == 1:
                self.mrefs[i] = ("q", self.store(qi))
            else:
                c, sn = g.sincos(qi, i)
                self.mrefs[i] = ("cs", self.store(c), self.store(sn))
        g.ty = "T"
        for i, v in qdv.items():
            self.qdrefs[i] = self.store(v)
        for key, v in xv.items():
            self.xrefs[key] = self.store(v)
        self.nprologue = self.nslot
        self.released = set()
        self.release_line = {}
        self.nphase = 0
        g.on_input = self._read_after_release
        for gi in sorted(g.groups_read):
            self.release(gi)

    def release(self, gi):
        """Every read of input group gi has been emitted: cx.fetch_next(gi)
        lets an asynchronous context start copying the next state's group gi
        into the buffer these reads came from (a no-op for the others).
        Emitted once per group; finish() releases whatever is left."""
        if gi in self.g.groups_read and gi not in self.released:
            self.released.add(gi)
            self.release_line[gi] = len(self.g.lines)
            self.g.raw(f"cx.fetch_next({gi});")

    def _read_after_release(self, gi):
        """A routine read group gi again after releasing it (OSC re-reads q
        for the posture torque): withdraw the early release; finish()
        releases the group after its last read."""
        if gi in self.released:
            self.released.discard(gi)
            self.g.lines[self.release_line.pop(gi)] = f"  // group {gi} is read again below: released at the end"

    def store(self, v):
        if isinstance(v, DualEx):  # value and tangent in their own slots
            return ("d", self.store(v.v), self.store(v.t))
        if v.c is not None:
            return ("k", v.c)
        k = self.nslot
        if self.g.ty == "TD":  # a double in two consecutive slots (one when T is double)
            self.nslot += 2
            self.g.raw(f"cx.st2({k}, {v.s});")
            return ("h", k)
        self.nslot += 1
        self.g.raw(f"cx.st({k}, {v.s});")
        return ("s", k)

    def load(self, ref):
        if ref[0] == "d":
            return DualEx(self.load(ref[1]), self.load(ref[2]))
        if ref[0] == "k":
            return K(ref[1])
        if ref[0] == "h":
            return self.g.tmp(f"cx.get2({ref[1]})", "r", ty="TD")
        return self.g.tmp(f"cx.get({ref[1]})", "r", ty="T")

    def joint(self, i):
        # a numbered phase point at every joint step: a kernel may barrier its
        # warps here so they walk the straight-line code together (I-cache reuse)
        self.g.raw(f"cx.template phase<{self.nphase}>();")
        self.nphase += 1
        m = self.mrefs[i]
        if m[0] == "q":
            return Joint(self.g, self.rb, i, q=self.load(m[1]))
        return Joint(self.g, self.rb, i, cs=(self.load(m[1]), self.load(m[2])))

    def gravity(self):
        # emitted once per routine (a fused routine runs several recursions)
        if getattr(self, "_gvec", None) is None:
            self.g.raw(f"const {self.g.ty} ga0 = cx.g(0), ga1 = cx.g(1), ga2 = cx.g(2);")
            self._gvec = [ZERO, ZERO, ZERO, Ex(s="ga0"), Ex(s="ga1"), Ex(s="ga2")]
        return self._gvec

    def finish(self):
        for gi in sorted(self.g.groups_read):
            self.release(gi)
        self.g.raw("return ok;")
        return self


def world_of(g, X, Wp):
    """World transform (R row-major 9, p 3) of joint X's body from its
    parent's (kinematics.hpp:43-56): local R = QO·QJ, p = tO + QO·tJ."""
    Rl = [g.dot(X.QO[3 * r:3 * r + 3], [X.QJ[c], X.QJ[3 + c], X.QJ[6 + c]]) for r in range(3) for c in range(3)]
    pl = g.vadd(X.tO, g.matvec(X.QO, X.tJ))
    if Wp is None:
        return Rl, pl
    R = [g.dot(Wp[0][3 * r:3 * r + 3], [Rl[c], Rl[3 + c], Rl[6 + c]]) for r in range(3) for c in range(3)]
    return R, g.vadd(g.matvec(Wp[0], pl), Wp[1])


def world_of_parent(g, X, W):
    """The parent's world transform rebuilt from the child's (W_p = W ∘ X⁻¹),
    so a DFS keeps only the current root->leaf transform live (as the
    velocities: v_p = X(v − S q̇))."""
    Rl = [g.dot(X.QO[3 * r:3 * r + 3], [X.QJ[c], X.QJ[3 + c], X.QJ[6 + c]]) for r in range(3) for c in range(3)]
    pl = g.vadd(X.tO, g.matvec(X.QO, X.tJ))
    Rp = [g.dot(W[0][3 * r:3 * r + 3], Rl[3 * c:3 * c + 3]) for r in range(3) for c in range(3)]  # R Rlᵀ
    return Rp, g.vsub(W[1], g.matvec(Rp, pl))


def fext_body(g, W, i):
    """External wrench on joint i (world Plücker about the origin, fext plane
    6i + k, ExternalForcesT dynamics.hpp:52-81) in body i coordinates:
    inverse_transform_force (spatial.hpp:249-254), n_b = Rᵀ(n − p × f), f_b = Rᵀ f."""
    fw = [g.tmp(f"cx.fx({6 * i + k})", "fx") for k in range(6)]
    R, p = W
    return g.matTvec(R, g.vsub(fw[:3], g.cross3(p, fw[3:]))) + g.matTvec(R, fw[3:])


def gen_aba(rb, hp=(), tau_prologue=False, dual=False, fext=False, A0=None, og=0):
    """ABA (Featherstone RBDA Table 7.1; oracle forward_dynamics,
    dynamics.hpp:421-444).  x(0) = q, x(1) = q̇, x(2) = τ; y(0, i) = q̈_i.

    Pass 1 and pass 2 run as one DFS (only the current root->leaf velocity is
    live; a parent's velocity is rebuilt from its child, v_p = X(v − S q̇));
    the pass-2 -> pass-3 state per joint (U/D, u/D) goes to slots.

    hp: joints whose steps are computed (and whose slots are stored) in double
    when T is float — mixed precision for the floating-base trunk, where the
    whole tree's articulated inertia is projected.

    fext: external wrenches (cx.fx, world Plücker, ExternalForcesT), applied
    as p^A_i = v×*Iv − ⁱX₀* f_i (RBDA Table 7.1; oracle aba_loop, subtracted
    like dynamics.hpp:243-245); the world transform rides the DFS like the
    velocity (forward on the way down, rebuilt from the child on the way up)."""
    # tau_prologue: τ loaded with q, q̇ up front into slots (faster for the
    # fp32 routine; for fp64 those 29 slots displace pass-2 state from shared
    # memory and it measured slower, so τ is read at each joint's pass-2 step)
    A = A0 or Algo(rb, True, hp, extra=(2,) if tau_prologue else (), dual=dual)
    g = A.g
    layout = {}


    def ty(i):
        g.ty = "TD" if i in A.hp else "T"

    def down_up(i, vp, Wp=None):
        ty(i)
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        v = X.S(qdi) if vp is None else g.vadd(X.motion_to_child(vp), X.S(qdi))
        W = world_of(g, X, Wp) if fext else None
        acc = None
        for c in rb.children[i]:
            (Ic, pc), v, W = down_up(c, v, W)
            acc = (Ic, pc) if acc is None else (g.ai_add(acc[0], Ic), g.vadd(acc[1], pc))
        ty(i)
        if rb.children[i]:  # re-read instead of keeping them live across the subtree
            X = A.joint(i)
            qdi = A.load(A.qdrefs[i])
        b = rb.rb(i)
        IA = g.ai_from_rb(b)
        pA = g.crf(v, g.rb_apply(b, v))
        if fext:
            pA = g.vsub(pA, fext_body(g, W, i))
        if acc is not None:
            IA = g.ai_add(IA, acc[0])
            pA = g.vadd(pA, acc[1])
        U = g.ai_apply(IA, X.Svec())
        D = X.Sdot(U)
        g.check_pos(D)
        dinv = g.recip(D)
        taui = A.load(A.xrefs[(2, i)]) if tau_prologue else g.input(2, i)
        u = g.sub(taui, X.Sdot(pA))
        Ud = [g.mul(x, dinv) for x in U]
        ud = g.mul(u, dinv)
        layout[i] = (A.store(ud), [A.store(x) for x in Ud])
        if vp is None:
            return None, None, None
        c = g.crm(v, X.S(qdi))
        ir, ic = (0, 1, 2, 0, 0, 1), (0, 1, 2, 1, 2, 2)  # Ia = IA − U Udᵀ
        Ia = {"A": [g.sub(IA["A"][k], g.mul(U[ir[k]], Ud[ic[k]])) for k in range(6)],
              "C": [g.sub(IA["C"][k], g.mul(U[3 + ir[k]], Ud[3 + ic[k]])) for k in range(6)],
              "B": [g.sub(IA["B"][3 * r + cc], g.mul(U[r], Ud[3 + cc])) for r in range(3) for cc in range(3)]}
        pa = g.vadd(g.vadd(pA, g.ai_apply(Ia, c)), [g.mul(x, ud) for x in U])
        vpar = X.motion_to_parent(g.vsub(v, X.S(qdi)))
        Wpar = world_of_parent(g, X, W) if fext else None
        return (X.ai_to_parent(Ia), X.force_to_parent(pa)), vpar, Wpar

    for r in rb.roots:
        down_up(r, None)
    A.release(2)  # τ is read only in pass 2
    ty(rb.roots[0])
    gvec = A.gravity()

    def down(i, vp, ap):
        ty(i)
        udr, Udr = layout[i]
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        if vp is None:
            v = X.S(qdi)
            a1 = X.motion_to_child(gvec)
        else:
            v = g.vadd(X.motion_to_child(vp), X.S(qdi))
            a1 = g.vadd(X.motion_to_child(ap), g.crm(v, X.S(qdi)))
        qdd = g.sub(A.load(udr), g.sdot([A.load(r) for r in Udr], a1))
        g.output(og, i, qdd)
        g.check_finite(qdd)
        if rb.children[i]:
            a = g.vadd(a1, X.S(qdd))
            for c in rb.children[i]:
                down(c, v, a)

    for r in rb.roots:
        down(r, None, None)
    return A.finish() if A0 is None else A


def gen_dyn(rb):
    """The fused forward-dynamics call (vd_dynamics; oracle crba +
    rnea(q, q̇, 0) + forward_dynamics, dynamics.hpp:330-444) as one routine:
    y(0, c·n + r) = M(r, c) (dense, as gen_crba), y(1, i) = bias c + g (as
    gen_rnea with q̈ = 0), y(2, i) = q̈ (as gen_aba).  The three recursions
    share one prologue (every joint's sin/cos and q̇ parked once) and one
    gravity read; x(2) = τ is read in the ABA's pass 2."""
    A = Algo(rb, True)
    gen_crba(rb, A0=A, og=0)
    gen_rnea(rb, True, False, A0=A, og=1)
    gen_aba(rb, A0=A, og=2)
    return A.finish()


def subtree(rb, c):
    out, stack = [], [c]
    while stack:
        i = stack.pop()
        out.append(i)
        stack.extend(rb.children[i])
    return sorted(out)


def gen_aba_role(rb, r):
    """One warp role of the branch-parallel ABA (small batches, where one
    thread's straight-line chain is the latency): the trunk (root .. the
    first branching joint s) and the subtree under s's child r.  Every role
    recomputes the trunk velocities, runs passes 1-2 on its subtree and
    publishes the subtree's articulated inertia and bias force in s's frame
    (cx.xput, 27 values); after a CTA barrier role 0 sums them, finishes
    pass 2 and runs pass 3 down the trunk, publishing s's acceleration; after
    a second barrier every role runs pass 3 on its subtree.  The arithmetic of
    every joint step is gen_aba's (RBDA Table 7.1)."""
    tr = trunk(rb)
    s_ = tr[-1]
    kids = rb.children[s_]
    R = len(kids)
    mine = subtree(rb, kids[r])
    A = Algo(rb, True, only=set(tr) | set(mine))
    g = A.g
    layout = {}

    def finish(i, v, acc):
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        b = rb.rb(i)
        IA = g.ai_from_rb(b)
        pA = g.crf(v, g.rb_apply(b, v))
        if acc is not None:
            IA = g.ai_add(IA, acc[0])
            pA = g.vadd(pA, acc[1])
        U = g.ai_apply(IA, X.Svec())
        D = X.Sdot(U)
        g.check_pos(D)
        dinv = g.recip(D)
        u = g.sub(g.input(2, i), X.Sdot(pA))
        Ud = [g.mul(x, dinv) for x in U]
        ud = g.mul(u, dinv)
        layout[i] = (A.store(ud), [A.store(x) for x in Ud])
        if rb.parent[i] < 0:
            return None, None
        c = g.crm(v, X.S(qdi))
        ir, ic = (0, 1, 2, 0, 0, 1), (0, 1, 2, 1, 2, 2)
        Ia = {"A": [g.sub(IA["A"][k], g.mul(U[ir[k]], Ud[ic[k]])) for k in range(6)],
              "C": [g.sub(IA["C"][k], g.mul(U[3 + ir[k]], Ud[3 + ic[k]])) for k in range(6)],
              "B": [g.sub(IA["B"][3 * rr + cc], g.mul(U[rr], Ud[3 + cc])) for rr in range(3) for cc in range(3)]}
        pa = g.vadd(g.vadd(pA, g.ai_apply(Ia, c)), [g.mul(x, ud) for x in U])
        vpar = X.motion_to_parent(g.vsub(v, X.S(qdi)))
        return (X.ai_to_parent(Ia), X.force_to_parent(pa)), vpar

    def down_up(i, vp):
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        v = X.S(qdi) if vp is None else g.vadd(X.motion_to_child(vp), X.S(qdi))
        acc = None
        for c in rb.children[i]:
            (Ic, pc), v = down_up(c, v)
            acc = (Ic, pc) if acc is None else (g.ai_add(acc[0], Ic), g.vadd(acc[1], pc))
        return finish(i, v, acc)

    def down(i, vp, ap, gvec=None):
        udr, Udr = layout[i]
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        if vp is None:
            v = X.S(qdi)
            a1 = X.motion_to_child(gvec)
        else:
            v = g.vadd(X.motion_to_child(vp), X.S(qdi))
            a1 = g.vadd(X.motion_to_child(ap), g.crm(v, X.S(qdi)))
        qdd = g.sub(A.load(udr), g.sdot([A.load(x) for x in Udr], a1))
        g.output(0, i, qdd)
        g.check_finite(qdd)
        return v, g.vadd(a1, X.S(qdd))

    # pass 1 down the trunk (every role)
    v = None
    for i in tr:
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        v = X.S(qdi) if v is None else g.vadd(X.motion_to_child(v), X.S(qdi))
    # passes 1-2 of the subtree, its contribution published in s's frame
    (Ic, pc), v_s = down_up(kids[r], v)
    vals = Ic["A"] + Ic["B"] + Ic["C"] + pc
    for k, x in enumerate(vals):
        g.raw(f"cx.xput({r * 27 + k}, {g.o(x)});")
    g.raw("cx.role_sync();")
    if r == 0:
        acc = None
        for rr in range(R):
            got = [g.tmp(f"cx.xget({rr * 27 + k})", "xg") for k in range(27)]
            c = ({"A": got[0:6], "B": got[6:15], "C": got[15:21]}, got[21:27])
            acc = c if acc is None else (g.ai_add(acc[0], c[0]), g.vadd(acc[1], c[1]))
        ret, vv = finish(s_, v_s, acc)
        for i in reversed(tr[:-1]):
            ret, vv = finish(i, vv, ret)
        A.release(2)
        gvec = A.gravity()
        vp = ap = None
        for i in tr:
            vp, ap = down(i, vp, ap, gvec)
        for k in range(6):
            g.raw(f"cx.xput({R * 27 + k}, {g.o(ap[k])});")
    A.release(2)
    g.raw("cx.role_sync();")
    a_s = [g.tmp(f"cx.xget({R * 27 + k})", "xa") for k in range(6)]

    def down_sub(i, vp, ap):
        vi, ai = down(i, vp, ap)
        for c in rb.children[i]:
            down_sub(c, vi, ai)

    down_sub(kids[r], v_s, a_s)
    return A.finish()


def gen_rnea(rb, with_qd, with_qdd, dual=False, fext=False, A0=None, og=0):
    """RNEA (rnea_loop, dynamics.hpp:272-327; Alg. 1 of PAPER.md:141-151):
    x(0) = q, x(1) = q̇ (if with_qd), x(2) = q̈ (if with_qdd); y(0, i) = τ_i.
    with_qdd = False is the bias term c + g (dynamics.hpp:434-435), with_qd =
    False as well the gravity term (dynamics.hpp:403-408).  One DFS: v, a and
    the body's own force on the way down, Σ child forces and τ on the way up.
    fext: f_i −= ⁱX₀* f_ext,i (dynamics.hpp:243-245, rnea_loop 316-318), the
    world transform carried down the DFS and rebuilt from the child between
    siblings."""
    A = A0 or Algo(rb, with_qd, extra=(2,) if with_qdd else (), dual=dual)
    g = A.g
    gvec = A.gravity()

    def rec(i, vp, ap, Wp=None):
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i]) if with_qd else ZERO
        qddi = A.load(A.xrefs[(2, i)]) if with_qdd else ZERO
        if vp is None:
            v = X.S(qdi)
            a = g.vadd(X.motion_to_child(gvec), X.S(qddi))
        else:
            v = g.vadd(X.motion_to_child(vp), X.S(qdi))
            a = g.vadd(g.vadd(X.motion_to_child(ap), g.crm(v, X.S(qdi))), X.S(qddi))
        b = rb.rb(i)
        f = g.vadd(g.rb_apply(b, a), g.crf(v, g.rb_apply(b, v)))
        W = None
        if fext:
            W = world_of(g, X, Wp)
            f = g.vsub(f, fext_body(g, W, i))
        for c in rb.children[i]:
            fc, W = rec(c, v, a, W)
            f = g.vadd(f, fc)
        if rb.children[i]:
            X = A.joint(i)
        tau = X.Sdot(f)
        g.output(og, i, tau)
        if vp is None:
            return None, None
        return X.force_to_parent(f), (world_of_parent(g, X, W) if fext else None)

    for r in rb.roots:
        rec(r, None, None)
    return A.finish() if A0 is None else A


def gen_crba(rb, dual=False, packed=False, A0=None, og=0):
    """CRBA (crba_loop, dynamics.hpp:369-400; Alg. 2 of PAPER.md:156-165):
    x(0) = q; y(0, c·n + r) = M(r, c), dense, with exact zeros between
    branches (dynamics.hpp:330-335, test_dynamics.cpp:200-216).  packed: only
    the branch-sparse lower triangle, y(0, k) = M(r_k, c_k) for the k-th pair
    of Robot.lower_pattern() (G1: 242 of 841 values).  Composite
    inertias (10-parameter form) are summed leaf -> root in one DFS; each
    column is emitted as soon as its composite is complete, walking the force
    F = Ic S up the ancestor chain."""
    A = A0 or Algo(rb, False, dual=dual)
    g = A.g
    n = rb.n
    related = [[False] * n for _ in range(n)]
    pidx = {rc: k for k, rc in enumerate(rb.lower_pattern())}

    def emit(r, c, val):
        related[r][c] = related[c][r] = True
        if packed:
            g.output(og, pidx[(r, c)], val)
            return
        g.output(og, c * n + r, val)
        if r != c:
            g.output(og, r * n + c, val)

    def rec(i):
        Ic = rb.rb(i)
        for c in rb.children[i]:
            cm, ch, cI = rec(c)
            Ic = (g.add(Ic[0], cm), g.vadd(Ic[1], ch), g.vadd(Ic[2], cI))
        X = A.joint(i)
        F = g.rb_apply(Ic, X.Svec())
        emit(i, i, X.Sdot(F))
        j = i
        while rb.parent[j] >= 0:
            F = A.joint(j).force_to_parent(F)
            j = rb.parent[j]
            emit(i, j, Joint_Sdot(g, rb, j, F))
        if rb.parent[i] < 0:
            return None
        return rb_to_parent(g, X, Ic)

    for r in rb.roots:
        rec(r)
    for c in range(n if not packed else 0):
        for r in range(n):
            if not related[r][c]:
                g.output(og, c * n + r, ZERO)
    return A.finish() if A0 is None else A


def Joint_Sdot(g, rb, j, f):
    ax = rb.axis(j)
    return g.dot(ax, f[3:] if rb.kind[j] == 1 else f[:3])


def rb_out(g, b, Q, t):
    """transform_inertia (spatial.hpp:259-267) on the 10-parameter form
    (vd_device.cuh rb_out): h' = Q h + m t, I' = Q I Qᵀ + (2 g·t + m|t|²) 1 − t uᵀ − g tᵀ."""
    m, h, I = b
    gq = g.matvec(Q, h)
    Ir = g.sym_rotate(Q, I)
    if all(x.is0() for x in t):
        return (m, gq, Ir)
    u = [g.add(gq[k], g.mul(m, t[k])) for k in range(3)]
    diag = g.add(g.dot(gq, t), g.dot(u, t))
    I2 = [g.add(Ir[k], g.sub(g.sub(diag, g.mul(t[k], u[k])), g.mul(gq[k], t[k]))) for k in range(3)]
    I2 += [g.sub(Ir[3], g.add(g.mul(t[0], u[1]), g.mul(gq[0], t[1]))),
           g.sub(Ir[4], g.add(g.mul(t[0], u[2]), g.mul(gq[0], t[2]))),
           g.sub(Ir[5], g.add(g.mul(t[1], u[2]), g.mul(gq[1], t[2])))]
    return (m, u, I2)


def rb_to_parent(g, X, b):
    return rb_out(g, rb_out(g, b, X.QJ, X.tJ), X.QO, X.tO)


def gen_fk(rb, dual=False):
    """forward_kinematics (kinematics.hpp:43-56): x(0) = q; y(0, 12 j + 3 c + r)
    = ⁰R_j(r, c) (column-major), y(0, 12 j + 9 + r) = ⁰p_j(r)."""
    A = Algo(rb, False, dual=dual)
    g = A.g

    def rec(i, Wp):
        X = A.joint(i)
        Rl = [g.dot(X.QO[3 * r:3 * r + 3], [X.QJ[c], X.QJ[3 + c], X.QJ[6 + c]]) for r in range(3) for c in range(3)]
        pl = g.vadd(X.tO, g.matvec(X.QO, X.tJ))
        if Wp is None:
            R, p = Rl, pl
        else:
            WR, Wpp = Wp
            R = [g.dot(WR[3 * r:3 * r + 3], [Rl[c], Rl[3 + c], Rl[6 + c]]) for r in range(3) for c in range(3)]
            p = g.vadd(g.matvec(WR, pl), Wpp)
        for c in range(3):
            for r in range(3):
                g.output(0, 12 * i + 3 * c + r, R[3 * r + c])
        for r in range(3):
            g.output(0, 12 * i + 9 + r, p[r])
        for c in rb.children[i]:
            rec(c, (R, p))

    for r in rb.roots:
        rec(r, None)
    return A.finish()


class Slots:
    """Named values kept in context slots (cx.st / cx.get): every write is a
    store (re-using the key's slot), every read a load.  Structural zeros
    stay symbolic constants and never touch a slot."""

    def __init__(self, A):
        self.A = A
        self.ref = {}

    def set(self, key, v):
        if v.c is not None:
            self.ref[key] = ("k", v.c)
            return
        old = self.ref.get(key)
        if old is not None and old[0] == "s":
            self.A.g.raw(f"cx.st({old[1]}, {v.s});")
        else:
            self.ref[key] = self.A.store(v)

    def get(self, key):
        return self.A.load(self.ref[key])


def chol6(g, G):
    """In-place Cholesky of a symmetric 6x6 (dict (r, c) -> Ex, lower), the
    same operation order as vd_algos.cuh chol6 / Eigen's LLT.  Returns (L, ok
    expression, pivots l_kk); L[(k, k)] holds the reciprocal 1 / l_kk, which
    is all the substitutions need (a multiply instead of an fp64 division per
    use: the divide is a ~10-instruction Newton sequence with a slow-path
    branch)."""
    L = dict(G)
    oks = []
    piv = []
    for k in range(6):
        x = L[(k, k)]
        for j in range(k):
            x = g.sub(x, g.mul(L[(k, j)], L[(k, j)]))
        oks.append(f"({g.o(x)} > T(0))")
        x = g.sqrt(x)
        piv.append(x)
        inv = g.recip(x, "iv")
        L[(k, k)] = inv
        for i in range(k + 1, 6):
            sv = L[(i, k)]
            for j in range(k):
                sv = g.sub(sv, g.mul(L[(i, j)], L[(k, j)]))
            L[(i, k)] = g.mul(sv, inv)
    return L, " && ".join(oks), piv


def chol6_solve(g, L, b):
    """L Lᵀ x = b with L from chol6 (reciprocal diagonal)."""
    b = list(b)
    for i in range(6):
        sv = b[i]
        for j in range(i):
            sv = g.sub(sv, g.mul(L[(i, j)], b[j]))
        b[i] = g.mul(sv, L[(i, i)])
    for i in range(5, -1, -1):
        sv = b[i]
        for j in range(i + 1, 6):
            sv = g.sub(sv, g.mul(L[(j, i)], b[j]))
        b[i] = g.mul(sv, L[(i, i)])
    return b


def gen_osc(rb, fj):
    """osc_step (control.hpp:108-155) for a task frame on joint fj (frame
    offset, target, gains, posture and ε are runtime parameters), mirroring
    vd_algos.cuh osc_one: CRBA -> M in compact ancestor rows, branch-sparse
    LTL (RBDA §6.5, no fill-in), M⁻¹ applied to the 6 Jacobian rows and the
    posture torque, Λ = (J M⁻¹ Jᵀ + εI)⁻¹ and (J M⁻¹ Jᵀ)⁻¹ by 6x6 Cholesky,
    τ = Jᵀ(F − z) + τ_post + c + g with the bias from RNEA.  Structural
    sparsity is symbolic: J is zero off the frame's ancestor path, so the
    Jacobian-row solves touch only that path.
    x(0) = q, x(1) = q̇; y(0, k) = τ_k, y(1, 6 c + r) = Λ(r, c)."""
    A = Algo(rb, True)
    g = A.g
    n = rb.n
    depth = [0] * n
    for i in range(n):
        depth[i] = 1 if rb.parent[i] < 0 else depth[rb.parent[i]] + 1
    path = []
    j = fj
    while j >= 0:
        path.append(j)
        j = rb.parent[j]
    path = path[::-1]  # root .. fj
    onpath = set(path)
    SL = Slots(A)

    # ---- frame pose along the path (kinematics.hpp:43-56, 89-96) and J (108-129)
    W = {}
    Wp = None
    for i in path:
        X = A.joint(i)
        Rl = [g.dot(X.QO[3 * r:3 * r + 3], [X.QJ[c], X.QJ[3 + c], X.QJ[6 + c]]) for r in range(3) for c in range(3)]
        pl = g.vadd(X.tO, g.matvec(X.QO, X.tJ))
        if Wp is None:
            R, p = Rl, pl
        else:
            R = [g.dot(Wp[0][3 * r:3 * r + 3], [Rl[c], Rl[3 + c], Rl[6 + c]]) for r in range(3) for c in range(3)]
            p = g.vadd(g.matvec(Wp[0], pl), Wp[1])
        W[i] = (R, p)
        Wp = (R, p)
    WR, Wpos = W[fj]
    fR = [g.tmp(f"cx.fR({k})", "pf") for k in range(9)]
    fpv = [g.tmp(f"cx.fp({k})", "pf") for k in range(3)]
    pose_R = [g.dot(WR[3 * r:3 * r + 3], [fR[c], fR[3 + c], fR[6 + c]]) for r in range(3) for c in range(3)]
    pose_p = g.vadd(g.matvec(WR, fpv), Wpos)
    for i in path:
        R, p = W[i]
        ax = g.matvec(R, rb.axis(i))
        if rb.kind[i] == 0:
            d = g.vsub(pose_p, p)
            col = ax + g.cross3(ax, d)
        else:
            col = [ZERO] * 3 + ax
        for r in range(6):
            SL.set(("J", r, i), col[r])
    # ---- pose error (control.hpp:73-77): log(R_t R_cᵀ), p_t − p_c
    tR = [g.tmp(f"cx.tR({k})", "pt") for k in range(9)]
    Rrel = [g.dot(tR[3 * r:3 * r + 3], pose_R[3 * c:3 * c + 3]) for r in range(3) for c in range(3)]
    rl = ", ".join(g.o(x) for x in Rrel)
    g.raw(f"const T Rrel_[9] = {{{rl}}};")
    g.raw("T lg_[3];")
    g.raw("vd_rotation_log(Rrel_, lg_);")
    err = [Ex(s="lg_[0]"), Ex(s="lg_[1]"), Ex(s="lg_[2]")]
    err += [g.sub(g.tmp(f"cx.tp({k})", "pt"), pose_p[k]) for k in range(3)]
    for k in range(6):
        SL.set(("err", k), err[k])

    # ---- CRBA (crba_loop, dynamics.hpp:369-400) into compact rows Mc(i, d) = M(i, anc_d(i))
    def crba(i):
        Ic = rb.rb(i)
        for c in rb.children[i]:
            cm, ch, cI = crba(c)
            Ic = (g.add(Ic[0], cm), g.vadd(Ic[1], ch), g.vadd(Ic[2], cI))
        X = A.joint(i)
        F = g.rb_apply(Ic, X.Svec())
        SL.set(("M", i, 0), X.Sdot(F))
        j, d = i, 0
        while rb.parent[j] >= 0:
            F = A.joint(j).force_to_parent(F)
            j = rb.parent[j]
            d += 1
            SL.set(("M", i, d), Joint_Sdot(g, rb, j, F))
        if rb.parent[i] < 0:
            return None
        return rb_to_parent(g, X, Ic)

    for r in rb.roots:
        crba(r)

    # ---- LTL in place (RBDA Table 6.3), k = n-1 .. 0
    def anc(i, d):
        for _ in range(d):
            i = rb.parent[i]
        return i

    for k in range(n - 1, -1, -1):
        dkk = SL.get(("M", k, 0))
        g.raw(f"ok = ok && ({g.o(dkk)} > T(0));")
        lkk = g.tmp(f"vd_sqrt({g.o(dkk)})", "sq")
        inv = g.tmp(f"T(1) / {lkk.s}", "iv")
        SL.set(("M", k, 0), inv)  # the substitutions below only need 1 / l_kk
        row = {0: lkk}
        for d in range(1, depth[k]):
            row[d] = g.mul(SL.get(("M", k, d)), inv)
            SL.set(("M", k, d), row[d])
        for d in range(1, depth[k]):
            i = anc(k, d)
            for e in range(d, depth[k]):
                SL.set(("M", i, e - d), g.sub(SL.get(("M", i, e - d)), g.mul(row[d], row[e])))

    # ---- 7 right-hand sides: rows of J and τ_post = kp_p (q_post − q) − kd_p q̇
    pkp, pkd = g.tmp("cx.pkp()", "pp"), g.tmp("cx.pkd()", "pp")

    def tpost(k):
        qk = g.input(0, k)
        return g.sub(g.mul(pkp, g.sub(g.tmp(f"cx.post({k})", "pp"), qk)), g.mul(pkd, A.load(A.qdrefs[k])))

    for k in range(n):
        for r in range(6):
            SL.set(("X", r, k), SL.get(("J", r, k)) if k in onpath else ZERO)
        SL.set(("X", 6, k), tpost(k))
    # Lᵀ y = b (leaf -> root), then L x = y (root -> leaf); only path entries of
    # x are needed (J is zero elsewhere)
    for i in range(n - 1, -1, -1):
        inv = SL.get(("M", i, 0))
        xi = {}
        for r in range(7):
            v = SL.get(("X", r, i)) if SL.ref[("X", r, i)][0] == "s" else K(SL.ref[("X", r, i)][1])
            xi[r] = g.mul(v, inv)
            SL.set(("X", r, i), xi[r])
        for d in range(1, depth[i]):
            j = anc(i, d)
            lij = None
            for r in range(7):
                if xi[r].is0():
                    continue
                if lij is None:
                    lij = SL.get(("M", i, d))
                cur = SL.get(("X", r, j)) if SL.ref[("X", r, j)][0] == "s" else K(SL.ref[("X", r, j)][1])
                SL.set(("X", r, j), g.sub(cur, g.mul(lij, xi[r])))
    xs = {}
    for i in path:
        acc = {r: (SL.get(("X", r, i)) if SL.ref[("X", r, i)][0] == "s" else K(SL.ref[("X", r, i)][1])) for r in range(7)}
        for d in range(1, depth[i]):
            j = anc(i, d)
            lij = SL.get(("M", i, d))
            for r in range(7):
                acc[r] = g.sub(acc[r], g.mul(lij, xs[(r, j)]))
        inv = SL.get(("M", i, 0))
        for r in range(7):
            xs[(r, i)] = g.mul(acc[r], inv)
    # ---- gram = J M⁻¹ Jᵀ, w = J M⁻¹ τ_post, J q̇
    Jp = {(r, k): SL.get(("J", r, k)) for r in range(6) for k in path}
    gram = {}
    for r in range(6):
        for c in range(r + 1):
            gram[(r, c)] = g.sum([g.mul(Jp[(r, k)], xs[(c, k)]) for k in path])
    w = [g.sum([g.mul(Jp[(r, k)], xs[(6, k)]) for k in path]) for r in range(6)]
    jqd = [g.sum([g.mul(Jp[(r, k)], A.load(A.qdrefs[k])) for k in path]) for r in range(6)]
    eps = g.tmp("cx.eps()", "pe")
    Gr = {key: (g.add(v, eps) if key[0] == key[1] else v) for key, v in gram.items()}
    Lr, _, _ = chol6(g, Gr)
    Lg, gok, _ = chol6(g, gram)
    g.raw(f"const bool gok_ = {gok};")
    F = [g.add(g.sub(g.mul(g.tmp(f"cx.kp({r})", "pg"), SL.get(("err", r))), g.mul(g.tmp(f"cx.kd({r})", "pg"), jqd[r])),
               g.tmp(f"cx.aff({r})", "pg")) for r in range(6)]
    F = chol6_solve(g, Lr, F)
    zg = chol6_solve(g, Lg, w)
    zr = chol6_solve(g, Lr, w)
    z = [g.tmp(f"gok_ ? {g.o(a)} : {g.o(b)}", "z") for a, b in zip(zg, zr)]
    fz = [g.sub(a, b) for a, b in zip(F, z)]
    jt = {k: g.sum([g.mul(Jp[(r, k)], fz[r]) for r in range(6)]) for k in path}
    for k in path:
        SL.set(("jt", k), jt[k])
    # ---- Λ = (J M⁻¹ Jᵀ + εI)⁻¹, column by column
    g.raw("if (cx.want_lambda()) {")
    for c in range(6):
        e = chol6_solve(g, Lr, [ONE if r == c else ZERO for r in range(6)])
        for r in range(6):
            g.raw(f"cx.y(1, {6 * c + r}, {g.o(e[r])});")
    g.raw("}")
    # ---- bias c + g (RNEA with q̈ = 0, dynamics.hpp:434-435) and τ
    gvec = A.gravity()

    def rec(i, vp, ap):
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        if vp is None:
            v = X.S(qdi)
            a = X.motion_to_child(gvec)
        else:
            v = g.vadd(X.motion_to_child(vp), X.S(qdi))
            a = g.vadd(X.motion_to_child(ap), g.crm(v, X.S(qdi)))
        b = rb.rb(i)
        f = g.vadd(g.rb_apply(b, a), g.crf(v, g.rb_apply(b, v)))
        for c in rb.children[i]:
            f = g.vadd(f, rec(c, v, a))
        if rb.children[i]:
            X = A.joint(i)
        tau = g.add(g.add(tpost(i), X.Sdot(f)), SL.get(("jt", i)) if i in onpath else ZERO)
        g.raw(f"cx.y(0, {i}, {g.o(tau)});")
        g.raw(f"ok = ok && vd_isfinite({g.o(tau)});")
        return X.force_to_parent(f) if vp is not None else None

    for r in rb.roots:
        rec(r, None, None)
    return A.finish()


def gen_osc_aba(rb, fj):
    """osc_step (control.hpp:108-155) for a task frame on joint fj through the
    articulated-body factorisation instead of M: the same quantities as
    gen_osc (Λ = (J M⁻¹ Jᵀ + εI)⁻¹, J M⁻¹ τ_post, c + g, τ) but M is never
    formed.  One ABA pass 2 at zero velocity and gravity over all joints
    (articulated inertias, with τ_post as the joint force) keeps U/D, 1/D
    and u/D of the path joints only; M⁻¹ τ_post and the six columns of the
    body-frame inverse task inertia G_b = J_b M⁻¹ J_bᵀ (a unit wrench at the
    frame body, propagated up the path and the accelerations back down it)
    are path-only sweeps; J never materialises: J = T J_b with
    T = [[R, 0], [−R [r_f]×, R]] (R the frame body's world rotation, r_f the
    frame point in body coordinates), so J M⁻¹ Jᵀ = T G_b Tᵀ, J q̇ = T v_b,
    and Jᵀ F is the body wrench Tᵀ F pushed up the path.  Per-state slot
    state is the prologue plus ~9 values per path joint, against the
    branch-sparse M of gen_osc (G1 `l_palm`: 486 -> ~220 slots), which is
    what bounds the G1 OSC (its L2 scratch slab spills to DRAM).
    Featherstone RBDA Table 7.1 (ABA with external forces: p^A = −f^x);
    the reference's LLT of M (control.hpp:131-149) is the oracle.
    x(0) = q, x(1) = q̇; y(0, k) = τ_k, y(1, 6 c + r) = Λ(r, c)."""
    A = Algo(rb, True)
    g = A.g
    path = []
    j = fj
    while j >= 0:
        path.append(j)
        j = rb.parent[j]
    path = path[::-1]  # root .. fj
    onpath = set(path)
    SL = Slots(A)

    # ---- world pose of the frame body (kinematics.hpp:43-56, 89-96)
    Wp = None
    for i in path:
        X = A.joint(i)
        Rl = [g.dot(X.QO[3 * r:3 * r + 3], [X.QJ[c], X.QJ[3 + c], X.QJ[6 + c]]) for r in range(3) for c in range(3)]
        pl = g.vadd(X.tO, g.matvec(X.QO, X.tJ))
        if Wp is None:
            Wp = (Rl, pl)
        else:
            Wp = ([g.dot(Wp[0][3 * r:3 * r + 3], [Rl[c], Rl[3 + c], Rl[6 + c]]) for r in range(3) for c in range(3)],
                  g.vadd(g.matvec(Wp[0], pl), Wp[1]))
    WR, Wpos = Wp
    fR = [g.tmp(f"cx.fR({k})", "pf") for k in range(9)]
    fpv = [g.tmp(f"cx.fp({k})", "pf") for k in range(3)]
    pose_R = [g.dot(WR[3 * r:3 * r + 3], [fR[c], fR[3 + c], fR[6 + c]]) for r in range(3) for c in range(3)]
    pose_p = g.vadd(g.matvec(WR, fpv), Wpos)
    for k in range(9):
        SL.set(("R", k), WR[k])
    # ---- pose error (control.hpp:73-77): log(R_t R_cᵀ), p_t − p_c
    tR = [g.tmp(f"cx.tR({k})", "pt") for k in range(9)]
    Rrel = [g.dot(tR[3 * r:3 * r + 3], pose_R[3 * c:3 * c + 3]) for r in range(3) for c in range(3)]
    g.raw(f"const T Rrel_[9] = {{{', '.join(g.o(x) for x in Rrel)}}};")
    g.raw("T lg_[3];")
    g.raw("vd_rotation_log(Rrel_, lg_);")
    err = [Ex(s="lg_[0]"), Ex(s="lg_[1]"), Ex(s="lg_[2]")]
    err += [g.sub(g.tmp(f"cx.tp({k})", "pt"), pose_p[k]) for k in range(3)]
    for k in range(6):
        SL.set(("err", k), err[k])

    pkp, pkd = g.tmp("cx.pkp()", "pp"), g.tmp("cx.pkd()", "pp")

    def tpost(k):  # τ_post = kp_p (q_post − q) − kd_p q̇ (control.hpp:150-151)
        qk = g.input(0, k)
        return g.sub(g.mul(pkp, g.sub(g.tmp(f"cx.post({k})", "pp"), qk)), g.mul(pkd, A.load(A.qdrefs[k])))

    # ---- ABA pass 2 at q̇ = 0, a_g = 0 with τ = τ_post (RBDA Table 7.1)
    def up(i):
        acc = None
        for c in rb.children[i]:
            Ic, pc = up(c)
            acc = (Ic, pc) if acc is None else (g.ai_add(acc[0], Ic), g.vadd(acc[1], pc))
        X = A.joint(i)
        IA = g.ai_from_rb(rb.rb(i))
        pA = [ZERO] * 6
        if acc is not None:
            IA = g.ai_add(IA, acc[0])
            pA = acc[1]
        U = g.ai_apply(IA, X.Svec())
        D = X.Sdot(U)
        g.check_pos(D)
        dinv = g.recip(D)
        u = g.sub(tpost(i), X.Sdot(pA))
        Ud = [g.mul(x, dinv) for x in U]
        ud = g.mul(u, dinv)
        if i in onpath:
            for k in range(6):
                SL.set(("Ud", i, k), Ud[k])
            SL.set(("dinv", i), dinv)
            SL.set(("ud", i), ud)
        if rb.parent[i] < 0:
            return None
        ir, ic = (0, 1, 2, 0, 0, 1), (0, 1, 2, 1, 2, 2)  # Ia = IA − U Udᵀ
        Ia = {"A": [g.sub(IA["A"][k], g.mul(U[ir[k]], Ud[ic[k]])) for k in range(6)],
              "C": [g.sub(IA["C"][k], g.mul(U[3 + ir[k]], Ud[3 + ic[k]])) for k in range(6)],
              "B": [g.sub(IA["B"][3 * r + cc], g.mul(U[r], Ud[3 + cc])) for r in range(3) for cc in range(3)]}
        pa = g.vadd(pA, [g.mul(x, ud) for x in U])
        return X.ai_to_parent(Ia), X.force_to_parent(pa)

    for r in rb.roots:
        up(r)

    def down_path(urefs):
        """Pass 3 down the path at zero velocity and gravity; urefs(i) -> u_i
        (or None: use the stored u/D).  Returns the frame body's acceleration."""
        a = None
        for i in path:
            X = A.joint(i)
            Ud = [SL.get(("Ud", i, k)) for k in range(6)]
            if a is not None:
                a = X.motion_to_child(a)
            u = urefs(i)
            qdd = SL.get(("ud", i)) if u is None else g.mul(u, SL.get(("dinv", i)))
            if a is not None:
                qdd = g.sub(qdd, g.sdot(Ud, a))
            a = X.S(qdd) if a is None else g.vadd(a, X.S(qdd))
        return a

    a_post = down_path(lambda i: None)  # M⁻¹ τ_post seen at the frame body
    apost = [g.tmp(g.o(x), "ap") if x.c is None else x for x in a_post]
    for k in range(6):
        SL.set(("apost", k), apost[k])

    # ---- G_b = J_b M⁻¹ J_bᵀ: unit wrench e_r at the frame body (p^A = −e_r)
    Gb = {}
    for r in range(6):
        pA = [K(-1.0) if k == r else ZERO for k in range(6)]
        for i in reversed(path):
            X = A.joint(i)
            u = g.neg(X.Sdot(pA))
            SL.set(("u", i), u)
            if rb.parent[i] >= 0:
                Ud = [SL.get(("Ud", i, k)) for k in range(6)]
                pA = X.force_to_parent(g.vadd(pA, [g.mul(x, u) for x in Ud]))
        col = down_path(lambda i: SL.get(("u", i)) if SL.ref[("u", i)][0] == "s" else K(SL.ref[("u", i)][1]))
        for k in range(6):
            Gb[(k, r)] = col[k]
            SL.set(("Gb", k, r), col[k])

    # ---- T = [[R, 0], [−R [r_f]×, R]]: body spatial vector -> world (ω, v at the frame point)
    R = [SL.get(("R", k)) for k in range(9)]
    rf = [g.tmp(f"cx.fp({k})", "pf") for k in range(3)]

    def Tm(m):
        return g.matvec(R, m[:3]) + g.matvec(R, g.vadd(m[3:], g.cross3(m[:3], rf)))

    TG = [Tm([SL.get(("Gb", k, c)) for k in range(6)]) for c in range(6)]  # TG[c] = column c of T G_b
    gram = {}
    for rr in range(6):
        row = Tm([TG[c][rr] for c in range(6)])  # row rr of T G_b Tᵀ
        for c in range(rr + 1):
            gram[(rr, c)] = row[c]
    w = Tm([SL.get(("apost", k)) for k in range(6)])
    # J q̇ = T v_b, v_b from the velocity pass down the path
    v = None
    for i in path:
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        v = X.S(qdi) if v is None else g.vadd(X.motion_to_child(v), X.S(qdi))
    jqd = Tm(v)
    eps = g.tmp("cx.eps()", "pe")
    Gr = {key: (g.add(val, eps) if key[0] == key[1] else val) for key, val in gram.items()}
    Lr, _, _ = chol6(g, Gr)
    Lg, gok, _ = chol6(g, gram)
    g.raw(f"const bool gok_ = {gok};")
    F = [g.add(g.sub(g.mul(g.tmp(f"cx.kp({r})", "pg"), SL.get(("err", r))), g.mul(g.tmp(f"cx.kd({r})", "pg"), jqd[r])),
               g.tmp(f"cx.aff({r})", "pg")) for r in range(6)]
    F = chol6_solve(g, Lr, F)
    zg = chol6_solve(g, Lg, w)
    zr = chol6_solve(g, Lr, w)
    z = [g.tmp(f"gok_ ? {g.o(a)} : {g.o(b)}", "z") for a, b in zip(zg, zr)]
    fz = [g.sub(a, b) for a, b in zip(F, z)]
    # ---- Jᵀ (F − z): body wrench Tᵀ fz = (Rᵀ n + r_f × Rᵀ f, Rᵀ f), pushed up the path
    fl = g.matTvec(R, fz[3:])
    fb = g.vadd(g.matTvec(R, fz[:3]), g.cross3(rf, fl)) + fl
    for i in reversed(path):
        X = A.joint(i)
        SL.set(("jt", i), X.Sdot(fb))
        if rb.parent[i] >= 0:
            fb = X.force_to_parent(fb)
    # ---- Λ = (J M⁻¹ Jᵀ + εI)⁻¹, column by column
    g.raw("if (cx.want_lambda()) {")
    for c in range(6):
        e = chol6_solve(g, Lr, [ONE if r == c else ZERO for r in range(6)])
        for r in range(6):
            g.raw(f"cx.y(1, {6 * c + r}, {g.o(e[r])});")
    g.raw("}")
    # ---- bias c + g (RNEA with q̈ = 0, dynamics.hpp:434-435) and τ
    gvec = A.gravity()

    def rec(i, vp, ap):
        X = A.joint(i)
        qdi = A.load(A.qdrefs[i])
        if vp is None:
            v = X.S(qdi)
            a = X.motion_to_child(gvec)
        else:
            v = g.vadd(X.motion_to_child(vp), X.S(qdi))
            a = g.vadd(X.motion_to_child(ap), g.crm(v, X.S(qdi)))
        b = rb.rb(i)
        f = g.vadd(g.rb_apply(b, a), g.crf(v, g.rb_apply(b, v)))
        for c in rb.children[i]:
            f = g.vadd(f, rec(c, v, a))
        if rb.children[i]:
            X = A.joint(i)
        tau = g.add(g.add(tpost(i), X.Sdot(f)), SL.get(("jt", i)) if i in onpath else ZERO)
        g.raw(f"cx.y(0, {i}, {g.o(tau)});")
        g.raw(f"ok = ok && vd_isfinite({g.o(tau)});")
        return X.force_to_parent(f) if vp is not None else None

    for r in rb.roots:
        rec(r, None, None)
    return A.finish()


def frame_pose_J(A, fj):
    """frame_transform + geometric_jacobian (kinematics.hpp:89-129) of the
    task frame on joint fj (offset cx.fR / cx.fp, row-major): pose (R
    row-major 9, p 3) and the Jacobian columns of the path joints (angular
    rows first; every other column is an exact zero)."""
    g, rb = A.g, A.rb
    path = []
    j = fj
    while j >= 0:
        path.append(j)
        j = rb.parent[j]
    path = path[::-1]
    W, Wp = {}, None
    for i in path:
        X = A.joint(i)
        Rl = [g.dot(X.QO[3 * r:3 * r + 3], [X.QJ[c], X.QJ[3 + c], X.QJ[6 + c]]) for r in range(3) for c in range(3)]
        pl = g.vadd(X.tO, g.matvec(X.QO, X.tJ))
        if Wp is None:
            R, p = Rl, pl
        else:
            R = [g.dot(Wp[0][3 * r:3 * r + 3], [Rl[c], Rl[3 + c], Rl[6 + c]]) for r in range(3) for c in range(3)]
            p = g.vadd(g.matvec(Wp[0], pl), Wp[1])
        W[i] = (R, p)
        Wp = (R, p)
    WR, Wpos = W[fj]
    fR = [g.tmp(f"cx.fR({k})", "pf") for k in range(9)]
    fpv = [g.tmp(f"cx.fp({k})", "pf") for k in range(3)]
    pose_R = [g.dot(WR[3 * r:3 * r + 3], [fR[c], fR[3 + c], fR[6 + c]]) for r in range(3) for c in range(3)]
    pose_p = g.vadd(g.matvec(WR, fpv), Wpos)
    J = {}
    for i in path:
        R, p = W[i]
        ax = g.matvec(R, rb.axis(i))
        col = (ax + g.cross3(ax, g.vsub(pose_p, p))) if rb.kind[i] == 0 else ([ZERO] * 3 + ax)
        for r in range(6):
            J[(r, i)] = col[r]
    return pose_R, pose_p, J, path


def _path(rb, fj):
    out = []
    while fj >= 0:
        out.append(fj)
        fj = rb.parent[fj]
    return set(out)


def gen_jac(rb, fj):
    """x(0) = q; y(0, ·) = frame pose (R column-major, p), y(1, 6 c + r) = J(r, c)."""
    A = Algo(rb, False, only=_path(rb, fj))
    g = A.g
    pose_R, pose_p, J, path = frame_pose_J(A, fj)
    for c in range(3):
        for r in range(3):
            g.raw(f"cx.y(0, {3 * c + r}, {g.o(pose_R[3 * r + c])});")
    for r in range(3):
        g.raw(f"cx.y(0, {9 + r}, {g.o(pose_p[r])});")
    for c in range(rb.n):
        for r in range(6):
            g.raw(f"cx.y(1, {6 * c + r}, {g.o(J.get((r, c), ZERO))});")
    return A.finish()


def _gram6(g, J, path, d):
    G = {}
    for r in range(6):
        for c in range(r + 1):
            v = g.sum([g.mul(J[(r, k)], J[(c, k)]) for k in path])
            G[(r, c)] = g.add(v, d) if (r == c and d is not None) else v
    return G


def gen_diffik(rb, fj):
    """diff_ik_step (control.hpp:79-97; vd_algos.cuh diffik_one): q̇ = Jᵀ (J Jᵀ
    + λ² I)⁻¹ (kp ⊙ err + twist_ff).  y(0, j) = q̇_j (zeroed by the kernel when
    the damped Gram matrix does not factor), y(1, r) = pose error."""
    A = Algo(rb, False, only=_path(rb, fj))
    g = A.g
    pose_R, pose_p, J, path = frame_pose_J(A, fj)
    tR = [g.tmp(f"cx.tR({k})", "pt") for k in range(9)]
    Rrel = [g.dot(tR[3 * r:3 * r + 3], pose_R[3 * c:3 * c + 3]) for r in range(3) for c in range(3)]
    g.raw(f"const T Rrel_[9] = {{{', '.join(g.o(x) for x in Rrel)}}};")
    g.raw("T lg_[3];")
    g.raw("vd_rotation_log(Rrel_, lg_);")
    err = [Ex(s="lg_[0]"), Ex(s="lg_[1]"), Ex(s="lg_[2]")]
    err += [g.sub(g.tmp(f"cx.tp({k})", "pt"), pose_p[k]) for k in range(3)]
    for r in range(6):
        g.raw(f"cx.y(1, {r}, {g.o(err[r])});")
    rhs = [g.add(g.mul(g.tmp(f"cx.kp({r})", "pg"), err[r]), g.tmp(f"cx.tw({r})", "pg")) for r in range(6)]
    lam = g.tmp("cx.damp()", "pd")
    L, okx, _ = chol6(g, _gram6(g, J, path, g.mul(lam, lam)))
    g.raw(f"ok = ok && {okx};")
    x = chol6_solve(g, L, rhs)
    for j in range(rb.n):
        v = g.sum([g.mul(J[(r, j)], x[r]) for r in range(6)]) if j in path else ZERO
        g.raw(f"cx.y(0, {j}, {g.o(v)});")
    return A.finish()


def gen_manip(rb, fj, dual=False):
    """manipulability (kinematics.hpp:138-153; vd_algos.cuh manip_one):
    sqrt(det(J Jᵀ)) as the product of the Cholesky pivots, 0 when it does not
    factor.  y(0, 0) = w.  dual: its JVP along the tangent input cx.dx(0, ·)
    (jvp_scalar, autodiff.hpp:52-62), y(1, 0) = D w · dq (0 where w is)."""
    A = Algo(rb, False, dual=dual, only=_path(rb, fj))
    g = A.g
    _, _, J, path = frame_pose_J(A, fj)
    L, okx, piv = chol6(g, _gram6(g, J, path, None))
    d = piv[0]
    for i in range(1, 6):
        d = g.mul(d, piv[i])
    g.raw(f"cx.y(0, 0, ({okx}) ? {g.o(d)} : T(0));")
    if dual:
        g.raw(f"cx.y(1, 0, ({okx}) ? {Gen.o(g, d.t)} : T(0));")
    return A.finish()


# (struct name, generator, output planes as a function of n, input groups)
def trunk(rb):
    """Root chain up to and including the first joint with several children
    (tree29: the six floating-base joints); empty for serial chains."""
    out, i = [], rb.roots[0] if rb.roots else -1
    while i >= 0:
        out.append(i)
        if len(rb.children[i]) != 1:
            break
        i = rb.children[i][0]
    return out if i >= 0 and len(rb.children[i]) > 1 else []


OPS = [("Aba", gen_aba, lambda rb: rb.n, 3),
       # fp32 kernels: the floating-base trunk in fp64 (DESIGN.md §Parity policy)
       ("AbaMixed", lambda rb: gen_aba(rb, trunk(rb), tau_prologue=True), lambda rb: rb.n, 3),
       ("Rnea", lambda rb: gen_rnea(rb, True, True), lambda rb: rb.n, 3),
       ("RneaBias", lambda rb: gen_rnea(rb, True, False), lambda rb: rb.n, 2),
       ("RneaGrav", lambda rb: gen_rnea(rb, False, False), lambda rb: rb.n, 1),
       # external wrenches (cx.fx planes): τ, bias and q̈ with f_ext (§8(f)3)
       ("RneaFext", lambda rb: gen_rnea(rb, True, True, fext=True), lambda rb: rb.n, 3),
       ("RneaBiasFext", lambda rb: gen_rnea(rb, True, False, fext=True), lambda rb: rb.n, 2),
       ("AbaFext", lambda rb: gen_aba(rb, fext=True), lambda rb: rb.n, 3),
       ("AbaMixedFext", lambda rb: gen_aba(rb, trunk(rb), tau_prologue=True, fext=True), lambda rb: rb.n, 3),
       ("Crba", gen_crba, lambda rb: rb.n * rb.n, 1),
       ("CrbaPacked", lambda rb: gen_crba(rb, packed=True), lambda rb: len(rb.lower_pattern()), 1),
       # forward-mode JVPs (autodiff.hpp:41-50 on dual.hpp scalars): value in
       # output group 0, tangent in group 1
       ("AbaJvp", lambda rb: gen_aba(rb, dual=True), lambda rb: rb.n, 3),
       ("RneaJvp", lambda rb: gen_rnea(rb, True, True, dual=True), lambda rb: rb.n, 3),
       ("CrbaJvp", lambda rb: gen_crba(rb, dual=True), lambda rb: rb.n * rb.n, 1),
       ("FkJvp", lambda rb: gen_fk(rb, dual=True), lambda rb: 12 * rb.n, 1),
       ("Fk", gen_fk, lambda rb: 12 * rb.n, 1)]


def emit(name, cls, rb):
    POOL.clear()
    body = emit_body(name, cls, rb, pool_ops=POOL_OPS.get(name, ()))
    import struct
    vals = sorted(POOL, key=lambda c: POOL[c])
    dv = ", ".join(float.hex(c) for c in vals) or "0.0"
    fv = ", ".join(float.hex(struct.unpack("<f", struct.pack("<f", c))[0]) + "f" for c in vals) or "0.0f"
    n = max(1, len(vals))
    # Constant pool (USE_POOL): one __constant__ table per robot, read with an
    # opaque ld.const per use so the compiler cannot hoist every constant of
    # the routine out of the persistent loop into registers.  C linkage: the
    # asm names the table; the header is included by one translation unit
    # per binary.
    # (table reads need no symbol name: internal linkage, no extern "C")
    if POOL_MODE == "asm":
        dev = [f'extern "C" {{ __constant__ double vd_kd_{name}[{n}] = {{{dv}}}; }}',
               f'extern "C" {{ __constant__ float vd_kf_{name}[{n}] = {{{fv}}}; }}']
    else:
        dev = [f"static __constant__ double vd_kd_{name}[{n}] = {{{dv}}};",
               f"static __constant__ float vd_kf_{name}[{n}] = {{{fv}}};"]
    pre = [f"// ---- {name}: {len(vals)} model constants",
           "#if defined(__CUDACC__)"] + dev + [
           "#endif",
           f"static const double vd_hkd_{name}[{n}] = {{{dv}}};",
           f"static const float vd_hkf_{name}[{n}] = {{{fv}}};"]
    kc = ["  template <class T, int I>",
          "  VD_HD static T kc() {",
          "#if defined(__CUDA_ARCH__)"] + ([
          f"    if constexpr (sizeof(T) == 8) return vd_kd_{name}[I]; else return vd_kf_{name}[I];"]
          if POOL_MODE != "asm" else [
          "    T v;",
          "    if constexpr (sizeof(T) == 8)",
          f'      asm volatile("ld.const.f64 %0, [vd_kd_{name}+%1];" : "=d"(v) : "n"(I * 8));',
          "    else",
          f'      asm volatile("ld.const.f32 %0, [vd_kf_{name}+%1];" : "=f"(v) : "n"(I * 4));',
          "    return v;"]) + [
          "#else",
          f"    if constexpr (sizeof(T) == 8) return vd_hkd_{name}[I]; else return vd_hkf_{name}[I];",
          "#endif",
          "  }"]
    if not POOL:  # literals only: no table, no accessor
        return body
    return pre + body[:4] + kc + body[4:]


# the routines a per-model JIT module carries (paper_2604_04310_b200/jit.py):
# the dynamics hot path; OSC, task-space and JVP calls stay on the loop kernels
JIT_OPS = ("Aba", "AbaMixed", "Rnea", "RneaBias", "RneaGrav", "RneaFext", "RneaBiasFext", "AbaFext", "AbaMixedFext",
           "Crba", "CrbaPacked", "Fk")


def emit_body(name, cls, rb, ops=None, tasks=True, task_joints=None, pool_ops=()):
    out = [f"// ---- {name}",
           f"struct Gen{cls} {{",
           f"  static constexpr int kN = {rb.n};",
           f"  static constexpr uint64_t kFingerprint = {rb.d['fp']:#x}ull;"]
    global _POOL_ON
    for op, fn, nout, nin in OPS:
        if ops is not None and op not in ops:
            continue
        _POOL_ON = op in pool_ops
        try:
            A = fn(rb)
        finally:
            _POOL_ON = False
        out += [f"  // {op}: {A.g.flops} mul/add after folding; {A.nslot} slots, the first {A.nprologue} written by the prologue",
                f"  struct {op} {{",
                f"    static constexpr int kSlots = {A.nslot};",
                f"    static constexpr int kDof = {rb.n};",
                f"    static constexpr int kPrologue = {A.nprologue};",
                f"    static constexpr int kFlops = {A.g.flops};",
                f"    static constexpr int kIn = {nin};",
                f"    static constexpr int kOut = {nout(rb)};",
                "    template <class T, class Cx>",
                "    VD_HD static bool run(Cx& cx) {"]
        out += ["    " + ln for ln in A.g.lines]
        out += ["    }", "  };"]
    # the fused M + bias + q̈ routine (vd_dynamics, config 3) for serial chains
    # of the builtin set (the branched G1 runs three launches: its fused state
    # would not fit on chip)
    if ops is None and all(p == i - 1 for i, p in enumerate(rb.parent)):
        A = gen_dyn(rb)
        out += [f"  // Dyn (M, bias, q̈): {A.g.flops} mul/add after folding; {A.nslot} slots",
                "  struct Dyn {",
                f"    static constexpr int kSlots = {A.nslot};",
                f"    static constexpr int kDof = {rb.n};",
                f"    static constexpr int kPrologue = {A.nprologue};",
                f"    static constexpr int kFlops = {A.g.flops};",
                "    static constexpr int kIn = 3;",
                f"    static constexpr int kOut = {rb.n * rb.n + 2 * rb.n};",
                "    template <class T, class Cx>",
                "    VD_HD static bool run(Cx& cx) {"]
        out += ["    " + ln for ln in A.g.lines]
        out += ["    }", "  };"]
    if not tasks:
        return out + ["};", ""]
    # OSC per task-frame joint (the frame offset stays a runtime parameter):
    # one variant for every leaf joint (end effectors) and the joints that
    # carry a named frame of the model
    osc_joints = sorted(set(i for i in range(rb.n) if not rb.children[i]) | set(rb.frame_joints))
    if task_joints is not None:
        osc_joints = sorted(set(task_joints))
    # branched trees: the articulated-body OSC (no M in per-state slots);
    # serial chains: M is small, the branch-sparse LTL form costs fewer flops
    serial = all(p == i - 1 for i, p in enumerate(rb.parent))
    for fj in osc_joints:
        _POOL_ON = "Osc" in pool_ops
        try:
            A = gen_osc(rb, fj) if serial else gen_osc_aba(rb, fj)
        finally:
            _POOL_ON = False
        out += [f"  // Osc on joint {fj}: {A.g.flops} mul/add after folding; {A.nslot} slots",
                f"  struct Osc{fj} {{",
                f"    static constexpr int kSlots = {A.nslot};",
                f"    static constexpr int kDof = {rb.n};",
                f"    static constexpr int kPrologue = {A.nprologue};",
                f"    static constexpr int kFlops = {A.g.flops};",
                "    static constexpr int kIn = 2;",
                f"    static constexpr int kOut = {rb.n};",
                "    template <class T, class Cx>",
                "    VD_HD static bool run(Cx& cx) {"]
        out += ["    " + ln for ln in A.g.lines]
        out += ["    }", "  };"]
    for fj in osc_joints:
        for nm, fn, nout in (("Jac", gen_jac, 12), ("DiffIk", gen_diffik, rb.n), ("Manip", gen_manip, 1),
                             ("ManipJvp", lambda rb, fj: gen_manip(rb, fj, dual=True), 1)):
            A = fn(rb, fj)
            out += [f"  // {nm} on joint {fj}: {A.g.flops} mul/add after folding; {A.nslot} slots",
                    f"  struct {nm}{fj} {{",
                    f"    static constexpr int kSlots = {A.nslot};",
                    f"    static constexpr int kDof = {rb.n};",
                    f"    static constexpr int kPrologue = {A.nprologue};",
                    f"    static constexpr int kFlops = {A.g.flops};",
                    "    static constexpr int kIn = 1;",
                    f"    static constexpr int kOut = {nout};",
                    "    template <class T, class Cx>",
                    "    VD_HD static bool run(Cx& cx) {"]
            out += ["    " + ln for ln in A.g.lines]
            out += ["    }", "  };"]
    out.append(f"  static constexpr int kOscJoints[] = {{{', '.join(str(j) for j in osc_joints)}}};")
    out.append("  // calls f(Jac<fj>{}, DiffIk<fj>{}, Manip<fj>{}, ManipJvp<fj>{}) for a generated frame joint;")
    out.append("  // false if none")
    out.append("  template <class F>")
    out.append("  static bool with_task(int fj, F&& f) {")
    out.append("    switch (fj) {")
    for fj in osc_joints:
        out.append(f"      case {fj}: f(Jac{fj}{{}}, DiffIk{fj}{{}}, Manip{fj}{{}}, ManipJvp{fj}{{}}); return true;")
    out.append("      default: return false;")
    out.append("    }")
    out.append("  }")
    out.append("  // calls f(Osc<fj>{}) for the generated variant of joint fj; false if none")
    out.append("  template <class F>")
    out.append("  static bool with_osc(int fj, F&& f) {")
    out.append("    switch (fj) {")
    for fj in osc_joints:
        out.append(f"      case {fj}: f(Osc{fj}{{}}); return true;")
    out.append("      default: return false;")
    out.append("    }")
    out.append("  }")
    out += ["};", ""]
    return out


def jit_source(lib, h, task_joints=(), cls="Jit"):
    """Translation unit of a per-model JIT module: the model's generated
    routines (JIT_OPS; with task_joints also OSC / Jacobian / diff-IK /
    manipulability on those frame joints) as struct Gen<cls>, then the C
    entry points of csrc/vd_jit_entry.cuh over them."""
    rb = Robot(packed_model(lib, h), frame_joints(lib, h))
    tj = sorted(set(task_joints))
    lines = ["// GENERATED at model load by paper_2604_04310_b200/jit.py; do not edit.",
             "#include \"vd_gen_launch.cuh\"", "", "namespace vdk {", ""]
    lines += emit_body(f"jit {rb.d['fp']:#x}", cls, rb, ops=JIT_OPS, tasks=bool(tj), task_joints=tj)
    lines += ["}  // namespace vdk", "", f"#define VD_JIT_ROBOT vdk::Gen{cls}"]
    if tj:
        lines += ["#define VD_JIT_TASKS 1"]
    lines += ["#include \"vd_jit_entry.cuh\"", ""]
    return "\n".join(lines), rb.d["fp"]


def emit_op(name, A, rb, nin, nout):
    """One generated routine as a struct with run<T>(Cx&)."""
    out = [f"  // {name}: {A.g.flops} mul/add after folding; {A.nslot} slots",
           f"  struct {name} {{",
           f"    static constexpr int kSlots = {A.nslot};",
           f"    static constexpr int kDof = {rb.n};",
           f"    static constexpr int kPrologue = {A.nprologue};",
           f"    static constexpr int kFlops = {A.g.flops};",
           f"    static constexpr int kIn = {nin};",
           f"    static constexpr int kOut = {nout};",
           "    template <class T, class Cx>",
           "    VD_HD static bool run(Cx& cx) {"]
    out += ["    " + ln for ln in A.g.lines]
    out += ["    }", "  };"]
    return out


def emit_roles(cls, rb):
    """struct Gen<cls>Roles: the branch-parallel ABA's warp roles (gen_aba_role)."""
    R = len(rb.children[trunk(rb)[-1]])
    out = [f"struct Gen{cls}Roles {{", f"  static constexpr int kRoles = {R};", f"  static constexpr int kN = {rb.n};"]
    for r in range(R):
        out += emit_op(f"Role{r}", gen_aba_role(rb, r), rb, 3, rb.n)
    return out + ["};", ""]
