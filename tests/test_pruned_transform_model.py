"""CPU model of the band-pruned fused transforms (paper_2601_00161_b200/csrc/
esp_fft.cu), restated in numpy and checked against full transforms.

The kernels keep only the in-band box after each 1D pass (x: kx <= band_x
as a half spectrum, y/z: |k| <= band), pack two real rows into one complex
FFT (x passes) and rebuild the real rows of the inverse from a
conjugate-symmetric extension with kx = 0 and Nyquist taken as real.  These
identities are what make the pruned pipeline exact; the GPU parity tests
check the kernels themselves.
"""

import numpy as np
import pytest


def fftfreq_int(M):
    return np.array([m if m < (M + 1) // 2 else m - M for m in range(M)])


def box(M, band):
    """In-band indices: nbx (x half spectrum) and the y/z index lists
    (esp_api.cu set_cell)."""
    nbx = min(band[0], M[0] // 2) + 1
    iy = [m for m, f in enumerate(fftfreq_int(M[1])) if abs(f) <= band[1]]
    iz = [m for m, f in enumerate(fftfreq_int(M[2])) if abs(f) <= band[2]]
    return nbx, np.array(iy), np.array(iz)


def x_r2c_pairs(rows, nbx):
    """P1: two real rows per complex FFT, split by Hermitian symmetry."""
    out = np.empty((rows.shape[0], nbx), dtype=complex)
    N = rows.shape[1]
    for r in range(0, rows.shape[0], 2):
        a = rows[r]
        b = rows[r + 1] if r + 1 < rows.shape[0] else np.zeros(N)
        Z = np.fft.fft(a + 1j * b)
        k = np.arange(nbx)
        Zk, Zm = Z[k], np.conj(Z[(N - k) % N])
        out[r] = 0.5 * (Zk + Zm)
        if r + 1 < rows.shape[0]:
            out[r + 1] = -0.5j * (Zk - Zm)
    return out


def x_c2r_pairs(cols, N):
    """P5: rows of nbx half-spectrum columns -> real rows (unnormalised)."""
    nb = cols.shape[1]
    out = np.empty((cols.shape[0], N))
    half = N // 2
    for r in range(0, cols.shape[0], 2):
        A = np.zeros(half + 1, dtype=complex)
        B = np.zeros(half + 1, dtype=complex)
        A[:nb] = cols[r]
        if r + 1 < cols.shape[0]:
            B[:nb] = cols[r + 1]
        A[0], A[half] = A[0].real, A[half].real
        B[0], B[half] = B[0].real, B[half].real
        Z = np.zeros(N, dtype=complex)
        Z[:half + 1] = A + 1j * B
        k = np.arange(1, half)
        Z[N - k] = np.conj(A[k]) + 1j * np.conj(B[k])
        z = np.fft.ifft(Z) * N
        out[r] = z.real
        if r + 1 < cols.shape[0]:
            out[r + 1] = z.imag
    return out


CASES = [((16, 12, 10), (3, 2, 4)), ((32, 24, 18), (7, 5, 4)), ((12, 16, 20), (6, 8, 10)),
         ((64, 48, 36), (20, 9, 17))]


@pytest.mark.parametrize("M,band", CASES)
def test_pruned_forward_equals_full_transform_on_the_box(M, band):
    rng = np.random.default_rng(sum(M))
    Mx, My, Mz = M
    grid = rng.standard_normal((Mz, My, Mx))          # [z][y][x]
    nbx, iy, iz = box(M, band)
    A = x_r2c_pairs(grid.reshape(Mz * My, Mx), nbx).reshape(Mz, My, nbx)     # P1
    B = np.fft.fft(A, axis=1)[:, iy, :]                                        # P2
    X = np.fft.fft(B, axis=0)[iz, :, :]                                        # P3
    full = np.fft.rfftn(grid, axes=(0, 1, 2))                                  # [kz][ky][kx]
    ref = full[np.ix_(iz, iy, np.arange(nbx))]
    assert np.max(np.abs(X - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("M,band", CASES)
def test_pruned_inverse_equals_full_inverse_of_the_masked_spectrum(M, band):
    rng = np.random.default_rng(7 + sum(M))
    Mx, My, Mz = M
    f = rng.standard_normal((Mz, My, Mx))
    F = np.fft.rfftn(f, axes=(0, 1, 2))
    nbx, iy, iz = box(M, band)
    keep = np.zeros(F.shape, dtype=bool)
    keep[np.ix_(iz, iy, np.arange(nbx))] = True
    Fm = np.where(keep, F, 0)
    ref = np.fft.irfftn(Fm, s=(Mz, My, Mx), axes=(0, 1, 2)) * (Mx * My * Mz)
    S = F[np.ix_(iz, iy, np.arange(nbx))]                       # box spectrum
    Zp = np.zeros((Mz, len(iy), nbx), dtype=complex)            # P3b: zero-padded z
    Zp[iz] = S
    C = np.fft.ifft(Zp, axis=0) * Mz
    Yp = np.zeros((Mz, My, nbx), dtype=complex)                 # P4: zero-padded y
    Yp[:, iy, :] = C
    D = np.fft.ifft(Yp, axis=1) * My
    out = x_c2r_pairs(D.reshape(Mz * My, nbx), Mx).reshape(Mz, My, Mx)   # P5
    assert np.max(np.abs(out - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_band_index_maps_match_the_kernels():
    """band_mode / band_index (esp_fft.cu): in-band index <-> mode."""
    for M in (8, 9, 32, 48, 96, 384):
        for b in (0, 1, 3, M // 2 - 1, M // 2, M):
            _, iy, _ = box((2, M, 2), (0, b, 0))
            nb = len(iy)
            mode = [bi if (nb == M or bi <= (nb - 1) // 2) else bi + M - nb for bi in range(nb)]
            assert list(iy) == mode
            for m in range(M):
                if nb == M:
                    idx = m
                else:
                    bb = (nb - 1) // 2
                    idx = m if m <= bb else (m - (M - nb) if m >= M - bb else -1)
                assert idx == (list(iy).index(m) if m in iy else -1)
