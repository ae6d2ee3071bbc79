"""Pins of the CPU oracle against things other than itself (CPU only).

Each test cites the passage that fixes the expected value.  A plausible slip
in oracle.c -- a dropped 1/2^n, a wrong Y phase sign, a transposed A, a wrong
bit order, a wrong k/m doubling rule -- fails at least the Kronecker brute
force (test_oracle_matches_kronecker_bruteforce) and usually several others.
"""
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
from tests.paulis import (LETTERS, all_strings, brute_force_coeffs, kron_string, reconstruct,
                          random_complex)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _parse_golden(path):
    blocks, cur = [], None
    with open(path) as f:
        for raw in f:
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            tok = line.split()
            if tok[0] == "matrix":
                cur = {"name": tok[1], "n": int(tok[2]), "rows": [], "coef": {}}
            elif tok[0] == "coef":
                cur["coef"][tok[1]] = complex(float(tok[2]), float(tok[3]))
            elif tok[0] == "end":
                blocks.append(cur)
                cur = None
            else:
                cur["rows"].append([complex(*map(float, e.split(","))) for e in tok])
    return blocks


# ---------------------------------------------------------------- PauliComposer
def test_compose_spec_examples():
    # SPEC.md l.72-74
    k, m, ny = oracle.compose("Z")
    assert list(k) == [0, 1] and list(m) == [1, -1] and ny == 0
    k, m, ny = oracle.compose("XZ")
    assert list(k) == [2, 3, 0, 1] and list(m) == [1, -1, 1, -1] and ny == 0
    k, m, ny = oracle.compose("Y")
    assert list(k) == [1, 0] and list(m) == [1, -1] and ny == 1


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_compose_matches_kronecker_exhaustive(n):
    # PAPER l.199-208 must reproduce the tensor product of l.37-55, entry by entry,
    # with P[j][k[j]] = (-i)^{n_Y mod 4} m[j] (l.184) and zeros elsewhere.
    N = 1 << n
    for s in all_strings(n):
        k, m, ny = oracle.compose(s)
        P = np.zeros((N, N), dtype=np.complex128)
        P[np.arange(N), k.astype(np.int64)] = ((-1j) ** (ny % 4)) * m
        assert np.array_equal(P, kron_string(s)), s


def test_compose_matches_kronecker_random_large():
    rng = np.random.default_rng(7)
    for n in (5, 6, 7):
        for _ in range(6):
            s = "".join(rng.choice(list(LETTERS), size=n))
            k, m, ny = oracle.compose(s)
            N = 1 << n
            P = np.zeros((N, N), dtype=np.complex128)
            P[np.arange(N), k.astype(np.int64)] = ((-1j) ** (ny % 4)) * m
            assert np.array_equal(P, kron_string(s)), s


# ---------------------------------------------------------------- coefficients
@pytest.mark.parametrize("n", [1, 2, 3])
def test_oracle_matches_kronecker_bruteforce(n):
    # alpha = Tr(P A)/2^n with dense Kronecker products, random complex A.
    rng = np.random.default_rng(100 + n)
    for _ in range(3):
        A = random_complex(rng, (1 << n, 1 << n))
        got = oracle.decompose(A)
        want = brute_force_coeffs(A)
        assert np.max(np.abs(got - want)) < 1e-13


def test_golden_spec_examples():
    for blk in _parse_golden(os.path.join(GOLDEN, "spec_examples.txt")):
        A = np.array(blk["rows"], dtype=np.complex128)
        n = blk["n"]
        got = oracle.decompose(A)
        for q, s in enumerate(all_strings(n)):
            want = blk["coef"].get(s, 0j)
            assert got[q] == want, (blk["name"], s, got[q], want)  # exact rationals
        # ordering convention: oracle q <-> text string
        assert [oracle.string_of(q, n) for q in range(4 ** n)] == all_strings(n)


@pytest.mark.parametrize("n", [1, 3, 5])
def test_identity_is_one_hot(n):
    got = oracle.decompose(np.eye(1 << n))
    assert got[0] == 1.0 and np.count_nonzero(got) == 1


@pytest.mark.parametrize("n", [1, 2, 4, 5])
def test_single_string_is_one_hot(n):
    rng = np.random.default_rng(n)
    for q0 in rng.integers(0, 4 ** n, size=4):
        s = oracle.string_of(int(q0), n)
        got = oracle.decompose(kron_string(s))
        assert got[q0] == 1.0 and np.count_nonzero(got) == 1, s


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_reconstruction(n):
    # A = sum_P alpha_P P (Theorem 1)
    rng = np.random.default_rng(200 + n)
    A = random_complex(rng, (1 << n, 1 << n))
    assert np.max(np.abs(reconstruct(oracle.decompose(A), n) - A)) < 1e-12


@pytest.mark.parametrize("n", [5, 7])
def test_parseval(n):
    # Orthogonality (Theorem 1, l.98-114): sum |alpha|^2 = ||A||_F^2 / 2^n
    rng = np.random.default_rng(300 + n)
    A = random_complex(rng, (1 << n, 1 << n))
    c = oracle.decompose(A)
    lhs = np.sum(np.abs(c) ** 2)
    rhs = np.sum(np.abs(A) ** 2) / (1 << n)
    assert abs(lhs - rhs) / rhs < 1e-13
    assert abs(oracle.frobenius2(A) - np.sum(np.abs(A) ** 2)) / rhs < 1e-12


@pytest.mark.parametrize("n", [1, 3, 6])
def test_diagonal_only_IZ_and_equals_hadamard(n):
    # Diagonal matrices decompose on {I,Z}^n only; on that set the
    # coefficients are the normalised Sylvester-Hadamard transform of the diagonal
    # (textbook special case, scipy.linalg.hadamard).
    rng = np.random.default_rng(400 + n)
    d = random_complex(rng, 1 << n)
    c = oracle.decompose(np.diag(d))
    strings = all_strings(n)
    iz = [q for q, s in enumerate(strings) if set(s) <= {"I", "Z"}]
    other = [q for q, s in enumerate(strings) if not set(s) <= {"I", "Z"}]
    assert np.all(c[other] == 0)
    H = scipy.linalg.hadamard(1 << n).astype(np.float64)
    want = H @ d / (1 << n)
    # {I,Z} string with Z at tensor position l <-> Hadamard row whose bit l is set
    z_of = [sum(1 << (n - 1 - p) for p, ch in enumerate(strings[q]) if ch == "Z") for q in iz]
    assert np.max(np.abs(c[iz] - want[z_of])) < 1e-13
    # diagonal accessor gives the same as dense storage
    assert np.array_equal(oracle.coeffs_diagonal(d, np.arange(4 ** n)), c)


@pytest.mark.parametrize("n", [2, 4, 5])
def test_hermitian_gives_real(n):
    # Theorem 2
    rng = np.random.default_rng(500 + n)
    B = random_complex(rng, (1 << n, 1 << n))
    c = oracle.decompose((B + B.conj().T) / 2)
    assert np.max(np.abs(c.imag)) < 1e-15 * 4 * n


@pytest.mark.parametrize("n", [2, 4])
def test_real_symmetric_odd_ny_vanish(n):
    # A real symmetric, P^T = (-1)^{n_Y} P  =>  alpha_P = 0 for odd n_Y (derived from
    # Tr(PA) = Tr((PA)^T)); alpha also real by Theorem 2.
    rng = np.random.default_rng(600 + n)
    B = rng.standard_normal((1 << n, 1 << n))
    c = oracle.decompose(B + B.T)
    for q, s in enumerate(all_strings(n)):
        if s.count("Y") % 2:
            assert abs(c[q]) < 1e-14
    assert np.max(np.abs(c.imag)) < 1e-14


def test_kronecker_factorisation_pins_order():
    # alpha(B (x) C) = alpha(B) (x) alpha(C) in text order: string s_B s_C.
    rng = np.random.default_rng(11)
    B = random_complex(rng, (4, 4))
    C = random_complex(rng, (8, 8))
    got = oracle.decompose(np.kron(B, C))
    want = np.kron(oracle.decompose(B), oracle.decompose(C))
    assert np.max(np.abs(got - want)) < 1e-13


def test_direct_sum():
    # A (+) B = I (x) (alpha+beta)/2 + Z (x) (alpha-beta)/2
    rng = np.random.default_rng(12)
    n = 3
    A = random_complex(rng, (8, 8))
    B = random_complex(rng, (8, 8))
    C = scipy.linalg.block_diag(A, B)
    c = oracle.decompose(C).reshape(4, 4 ** n)   # leading letter I, X, Y, Z
    a, b = oracle.decompose(A), oracle.decompose(B)
    assert np.max(np.abs(c[0] - (a + b) / 2)) < 1e-14
    assert np.max(np.abs(c[3] - (a - b) / 2)) < 1e-14
    assert np.all(c[1] == 0) and np.all(c[2] == 0)


def test_hermitian_augmentation():
    # [[0, A^*],[A, 0]] = X (x) Re(alpha) + Y (x) Im(alpha)
    rng = np.random.default_rng(13)
    A = random_complex(rng, (8, 8))
    aug = np.block([[np.zeros((8, 8)), A.conj().T], [A, np.zeros((8, 8))]])
    c = oracle.decompose(aug).reshape(4, 64)
    a = oracle.decompose(A)
    assert np.max(np.abs(c[1] - a.real)) < 1e-14
    assert np.max(np.abs(c[2] - a.imag)) < 1e-14
    assert np.all(c[0] == 0) and np.all(c[3] == 0)


def test_linearity():
    # PAPER l.574-576
    rng = np.random.default_rng(14)
    A = random_complex(rng, (16, 16))
    B = random_complex(rng, (16, 16))
    mu = 0.3 - 1.7j
    got = oracle.decompose(mu * A + B)
    want = mu * oracle.decompose(A) + oracle.decompose(B)
    assert np.max(np.abs(got - want)) < 1e-13


def test_adjoint_and_transpose_relations():
    # alpha(A^H) = conj(alpha(A)) (P Hermitian); alpha(A^T)_P = (-1)^{n_Y} alpha(A)_P
    rng = np.random.default_rng(15)
    A = random_complex(rng, (16, 16))
    a = oracle.decompose(A)
    assert np.max(np.abs(oracle.decompose(A.conj().T) - a.conj())) < 1e-14
    sign = np.array([(-1) ** s.count("Y") for s in all_strings(4)])
    assert np.max(np.abs(oracle.decompose(A.T) - sign * a)) < 1e-14


# ---------------------------------------------------------------- structure theorems
def _tridiag(rng, n):
    N = 1 << n
    return (np.diag(random_complex(rng, N)) + np.diag(random_complex(rng, N - 1), 1)
            + np.diag(random_complex(rng, N - 1), -1))


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_tridiagonal_term_count(n):
    # Theorem and Table I (l.513): at most (n+1) 2^n terms;
    # for generic complex data exactly that many.
    rng = np.random.default_rng(700 + n)
    c = oracle.decompose(_tridiag(rng, n))
    nz = np.count_nonzero(np.abs(c) > 1e-14)
    assert nz == (n + 1) * (1 << n)


def test_tridiagonal_support_n2_spec():
    # support = {II,IZ,ZI,ZZ, IX,IY,ZX,ZY, XX,XY,YX,YY}
    rng = np.random.default_rng(8)
    c = oracle.decompose(_tridiag(rng, 2))
    sup = {s for q, s in enumerate(all_strings(2)) if abs(c[q]) > 1e-14}
    assert sup == {"II", "IZ", "ZI", "ZZ", "IX", "IY", "ZX", "ZY", "XX", "XY", "YX", "YY"}


@pytest.mark.parametrize("s", [1, 2, 3])
@pytest.mark.parametrize("n", [3, 4, 5])
def test_band_term_bound(s, n):
    # Band theorem: at most (s n - c(s)) 2^n terms,
    # c(s) = s(floor(log2 s)+1) - 2^{floor(log2 s)+1}.
    if (1 << n) <= s:
        pytest.skip("band wider than matrix")
    rng = np.random.default_rng(800 + 10 * n + s)
    N = 1 << n
    A = np.zeros((N, N), dtype=np.complex128)
    for dd in range(-s, s + 1):
        A += np.diag(random_complex(rng, N - abs(dd)), dd)
    L = int(np.floor(np.log2(s)))
    cs = s * (L + 1) - (1 << (L + 1))
    nz = np.count_nonzero(np.abs(oracle.decompose(A)) > 1e-14)
    assert nz <= (s * n - cs) * N


# ---------------------------------------------------------------- accessors / sampling
def test_sampled_coeffs_match_full():
    rng = np.random.default_rng(16)
    A = random_complex(rng, (64, 64))
    full = oracle.decompose(A)
    qs = rng.integers(0, 4 ** 6, size=100).astype(np.uint64)
    assert np.array_equal(oracle.coeffs_dense(A, qs), full[qs])


def test_tridiagonal_accessor_matches_dense():
    import ptdr_inputs

    n = 5
    sub, main, sup = ptdr_inputs.band(n, 3, "tridiagonal")
    A = ptdr_inputs.densify_band(n, main, sub, sup)
    qs = np.arange(4 ** n, dtype=np.uint64)
    assert np.array_equal(oracle.coeffs_tridiagonal(sub, main, sup, qs), oracle.decompose(A))


def test_generated_accessor_matches_dense():
    import ptdr_inputs

    n = 5
    for v in (ptdr_inputs.GENERAL, ptdr_inputs.HERMITIAN, ptdr_inputs.REAL_SYMMETRIC):
        A = ptdr_inputs.dense(n, 4, v)
        qs = np.arange(0, 4 ** n, 7, dtype=np.uint64)
        assert np.array_equal(oracle.coeffs_generated(n, 4, v, qs), oracle.coeffs_dense(A, qs))


# ---------------------------------------------------------------- anti-diagonal, band(s)
def _band_storage(rng, n, s):
    """diags[d + s][i] = A[i][i + d] and the dense matrix it stands for."""
    N = 1 << n
    diags = random_complex(rng, (2 * s + 1, N))
    A = np.zeros((N, N), dtype=np.complex128)
    for d in range(-s, s + 1):
        for i in range(N):
            if 0 <= i + d < N:
                A[i, i + d] = diags[d + s, i]
    return diags, A


@pytest.mark.parametrize("n", [1, 2, 3])
def test_antidiagonal_accessor_matches_kronecker(n):
    # anti-diagonal remark: A[i][2^n-1-i] only
    rng = np.random.default_rng(900 + n)
    N = 1 << n
    a = random_complex(rng, N)
    A = np.zeros((N, N), dtype=np.complex128)
    A[np.arange(N), N - 1 - np.arange(N)] = a
    got = oracle.coeffs_antidiagonal(a, np.arange(4 ** n, dtype=np.uint64))
    assert np.max(np.abs(got - brute_force_coeffs(A))) < 1e-14


@pytest.mark.parametrize("n", [2, 4, 6])
def test_antidiagonal_only_XY_strings(n):
    # l.391-392: "swap I,Z <-> X,Y" of the diagonal case -- only {X,Y}^n strings, 2^n of them
    rng = np.random.default_rng(910 + n)
    a = random_complex(rng, 1 << n)
    c = oracle.coeffs_antidiagonal(a, np.arange(4 ** n, dtype=np.uint64))
    for q in np.nonzero(np.abs(c) > 1e-14)[0]:
        assert set(oracle.string_of(int(q), n)) <= {"X", "Y"}
    assert np.count_nonzero(np.abs(c) > 1e-14) == 1 << n


@pytest.mark.parametrize("s,n", [(1, 3), (2, 3), (3, 2)])
def test_band_accessor_matches_kronecker(s, n):
    rng = np.random.default_rng(920 + 10 * s + n)
    diags, A = _band_storage(rng, n, s)
    got = oracle.coeffs_band(diags, s, np.arange(4 ** n, dtype=np.uint64))
    assert np.max(np.abs(got - brute_force_coeffs(A))) < 1e-13


@pytest.mark.parametrize("s,n", [(1, 5), (2, 5), (3, 5), (4, 6), (5, 6), (8, 6)])
def test_band_xmask_set_and_count(s, n):
    # Band theorem (Table I l.500-518): the nonzero X-masks are those of
    # the 2s+1 diagonals, x in {0} U {i ^ (i+d)}, and there are s n - c(s) of them
    # (equality verified for generic data).
    rng = np.random.default_rng(940 + 10 * s + n)
    diags, A = _band_storage(rng, n, s)
    c = oracle.coeffs_band(diags, s, np.arange(4 ** n, dtype=np.uint64))
    xs = set()
    for q in np.nonzero(np.abs(c) > 1e-14)[0]:
        x = 0
        for l in range(n):
            code = (int(q) >> (2 * l)) & 3
            x |= (1 if code in (1, 2) else 0) << l
        xs.add(x)
    N = 1 << n
    want = {0} | {i ^ (i + d) for d in range(1, s + 1) for i in range(N - d)}
    assert xs == want
    L = int(np.floor(np.log2(s)))
    cs = s * (L + 1) - (1 << (L + 1))
    assert len(want) == s * n - cs


# ---- the oracle's compensated trace (R7: mandatory at n >= 16) ---------------------
def test_neumaier_trace_small_exact():
    """Tr of diag(1, 1e16, 1, -1e16) is 2: plain left-to-right double summation returns 0
    (1e16 + 1 rounds to 1e16), a dropped compensation term returns 0, and swapping the two
    branches of the compensation update loses a unit as well.  The oracle must give the
    exact 2 / 2^n for II and IZ (z = 1: signs +,-,+,- of the same entries in reverse)."""
    d = np.array([1.0, 1e16, 1.0, -1e16])
    assert ((1.0 + 1e16) + 1.0) - 1e16 == 0.0  # the naive sum of the same order fails
    out = oracle.decompose(np.diag(d).astype(np.complex128))
    assert out[0] == 0.5                        # II: (1 + 1e16 + 1 - 1e16) / 4
    d2 = np.array([1.0, -1e16, 1.0, 1e16])      # IZ trace: 1 + 1e16 + 1 - 1e16 with signs folded in
    out2 = oracle.decompose(np.diag(d2).astype(np.complex128))
    assert out2[3] == 0.5
    # the imaginary accumulator is compensated too
    out3 = oracle.decompose(np.diag(1j * d).astype(np.complex128))
    assert out3[0] == 0.5j


def test_neumaier_trace_adversarial_2pow16():
    """A 2^16-term trace whose partial sums reach ~1e18 while the exact total (checked with
    fractions.Fraction) is the sum of the small terms alone: naive summation loses all of
    them, the oracle's Neumaier sum stays within the compensated bound n u^2 sum|x|."""
    from fractions import Fraction

    n = 16
    N = 1 << n
    rng = np.random.default_rng(1616)

    def adversarial():
        big = rng.integers(1, 1 << 20, N // 4).astype(np.float64) * 2.0 ** 33   # ~1e16
        big *= rng.choice([-1.0, 1.0], big.size)
        small = rng.random(N // 2)
        # first half: +big interleaved with small terms; second half: -big (shuffled)
        # interleaved with small terms -> the bigs cancel exactly in the true sum
        first = np.empty(N // 2)
        first[0::2], first[1::2] = big, small[: N // 4]
        second = np.empty(N // 2)
        second[0::2], second[1::2] = -rng.permutation(big), small[N // 4:]
        return np.concatenate([first, second])

    re, im = adversarial(), adversarial()
    exact_re = sum(Fraction(float(v)) for v in re)
    exact_im = sum(Fraction(float(v)) for v in im)
    naive_re = 0.0
    for v in re:
        naive_re += v
    bound_re = N * (2.0 ** -53) ** 2 * float(np.sum(np.abs(re))) + 2.0 ** -52 * abs(float(exact_re))
    bound_im = N * (2.0 ** -53) ** 2 * float(np.sum(np.abs(im))) + 2.0 ** -52 * abs(float(exact_im))
    assert abs(naive_re - float(exact_re)) > 1e3 * bound_re   # the input defeats plain summation
    got = oracle.coeffs_diagonal(re + 1j * im, np.array([0], dtype=np.uint64))[0] * N
    assert abs(Fraction(got.real) - exact_re) <= Fraction(bound_re)
    assert abs(Fraction(got.imag) - exact_im) <= Fraction(bound_im)
