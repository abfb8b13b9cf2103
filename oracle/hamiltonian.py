"""CPU restatement of the molecular-Hamiltonian path (TEST INFRASTRUCTURE ONLY).

Restates /root/reference/pkg/src/irlnqs/hamiltonian.py (``ham``) and the
excitation sign of hilbert.py for small cases, in plain Python over integer
bitmasks:

* ``matrix_element``            ham:180-235 (Slater-Condon, chemists' g)
* ``connected``                 ham:238-287 (singles + doubles, drop tolerance,
                                 ascending partner order, diagonal first)
* ``local_energy``              ham:290-302
* ``dense_hamiltonian``         ham:305-339 (explicit sector matrix)

Pinned to the reference's own outputs by tests/golden/hamiltonian.npz
(oracle/make_golden.py); the device path is checked against both.
"""

from __future__ import annotations

from itertools import combinations

import numpy as np

DROP = 1e-14


def _spatial(i, half):
    return i if i < half else i - half


def _same(i, j, half):
    return (i < half) == (j < half)


def _occ(bits, m):
    return [i for i in range(m) if (bits >> i) & 1]


def move_sign(bits, hole, part):
    """hilbert.py:126-134: parity of the occupied orbitals strictly between."""
    lo, hi = min(hole, part), max(hole, part)
    mask = ((1 << hi) - 1) ^ ((1 << (lo + 1)) - 1)
    return -1 if bin(bits & mask).count("1") % 2 else 1


def excitation(x, y, m):
    """hilbert.py:137-158: (degree, holes, particles, sign) taking x to y."""
    diff = x ^ y
    deg = bin(diff).count("1") // 2
    holes = [i for i in range(m) if (diff >> i) & 1 and (x >> i) & 1]
    parts = [i for i in range(m) if (diff >> i) & 1 and (y >> i) & 1]
    if deg == 0:
        return 0, [], [], 1
    if deg > 2 or len(holes) != len(parts):
        return deg, holes, parts, 1
    sign, bits = 1, x
    for h, p in zip(holes, parts):
        sign *= move_sign(bits, h, p)
        bits = (bits & ~(1 << h)) | (1 << p)
    return deg, holes, parts, sign


def matrix_element(e_core, h, g, x, y, ns):
    """<y|H|x> (ham:180-235)."""
    m = 2 * ns
    deg, holes, parts, sign = excitation(x, y, m)
    if deg == 0:
        occ = _occ(x, m)
        val = e_core + sum(h[_spatial(i, ns), _spatial(i, ns)] for i in occ)
        for a, i in enumerate(occ):
            si = _spatial(i, ns)
            for j in occ[a + 1:]:
                sj = _spatial(j, ns)
                val += g[si, si, sj, sj]
                if _same(i, j, ns):
                    val -= g[si, sj, sj, si]
        return val
    if deg == 1:
        a, p = holes[0], parts[0]
        if not _same(a, p, ns):
            return 0.0
        sa, sp = _spatial(a, ns), _spatial(p, ns)
        val = h[sa, sp]
        for j in _occ(x, m):
            if j == a:
                continue
            sj = _spatial(j, ns)
            val += g[sa, sp, sj, sj]
            if _same(a, j, ns):
                val -= g[sa, sj, sj, sp]
        return sign * val
    if deg == 2:
        (a, b), (p, q) = holes, parts
        sa, sb, sp, sq = (_spatial(i, ns) for i in (a, b, p, q))
        direct = g[sa, sp, sb, sq] if _same(a, p, ns) and _same(b, q, ns) else 0.0
        cross = g[sa, sq, sb, sp] if _same(a, q, ns) and _same(b, p, ns) else 0.0
        return sign * (direct - cross)
    return 0.0


def connected(e_core, h, g, x, ns, drop=DROP):
    """ham:238-287: [(x, diag)] + kept partners in ascending bitmask order."""
    m = 2 * ns
    occ = _occ(x, m)
    up_o = [i for i in occ if i < ns]
    dn_o = [i for i in occ if i >= ns]
    up_v = [i for i in range(ns) if not (x >> i) & 1]
    dn_v = [i for i in range(ns, m) if not (x >> i) & 1]
    ys = []
    for ho, vi in ((up_o, up_v), (dn_o, dn_v)):
        ys += [(x & ~(1 << a)) | (1 << p) for a in ho for p in vi]
    for ho, vi in ((up_o, up_v), (dn_o, dn_v)):
        for a, b in combinations(ho, 2):
            for p, q in combinations(vi, 2):
                ys.append((x & ~(1 << a) & ~(1 << b)) | (1 << p) | (1 << q))
    for a in up_o:
        for b in dn_o:
            for p in up_v:
                for q in dn_v:
                    ys.append((x & ~(1 << a) & ~(1 << b)) | (1 << p) | (1 << q))
    out = [(x, matrix_element(e_core, h, g, x, x, ns))]
    for y in sorted(ys):
        el = matrix_element(e_core, h, g, x, y, ns)
        if abs(el) > drop:
            out.append((y, el))
    return out


def local_energy(logpsi, e_core, h, g, x, ns):
    """ham:290-302: sum over the connected entries of element * psi(y)/psi(x)."""
    lx = complex(logpsi(x))
    return sum(el * np.exp(complex(logpsi(y)) - lx) for y, el in connected(e_core, h, g, x, ns))


def dense_hamiltonian(e_core, h, g, configs, ns):
    """ham:305-339 on a list of sector bitmasks."""
    idx = {c: k for k, c in enumerate(configs)}
    mat = np.zeros((len(configs), len(configs)))
    for k, x in enumerate(configs):
        for y, el in connected(e_core, h, g, x, ns, drop=0.0):
            if y in idx:
                mat[idx[y], k] = el
    return mat


def random_fcidump(seed, ns, n_elec, ms2=0, scale=0.3):
    """Seeded synthetic FCIDUMP text (input generator; lives with the other
    synthetic inputs in paper_2601_01437_b200/synthetic.py)."""
    from paper_2601_01437_b200.synthetic import molecule_fcidump

    return molecule_fcidump(seed, ns, n_elec, ms2=ms2, scale=scale)
