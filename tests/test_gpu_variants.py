"""The kernel variants selected by heuristics (or only by environment switches) must give the
same parity: Jacobi rounds on 2- and 4-CTA clusters and with 16-column blocks, the 64x64 /
64x48 GEMM tiles, the unscaled Cholesky, the Jacobi sweep replayed as a CUDA graph, the persistent (one cooperative launch per SVD) and
launch-per-round Jacobi sweeps, the compressed operator from a warm-started, a single or a double CholQR pass, the 8- and 16-byte SpMM, the segmented (gather) SpMM, the tiled and the entry-parallel SDDMM (the slab kernels' fallbacks)
under the factored operator. Each variant runs in a child process (the switches are
read once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [
    {"DFCG_JACOBI_CLUSTER": "2"},
    {"DFCG_JACOBI_CLUSTER": "4"},
    {"DFCG_JACOBI_NB": "16"},
    {"DFCG_JACOBI_NB": "16", "DFCG_JACOBI_CLUSTER": "2"},
    {"DFCG_GEMM_VARIANT": "4"},
    {"DFCG_GEMM_VARIANT": "7"},
    {"DFCG_CHOL_SCALE": "0"},
    {"DFCG_JACOBI_GRAPH": "1"},
    {"DFCG_PDL": "2"},
    {"DFCG_CHOL_INV_LATE": "0", "DFCG_CHOL_FUSED": "0"},
    {"DFCG_CHOL_FUSED": "0"},
    {"DFCG_PDL": "0", "DFCG_JACOBI_PDL": "0"},
    {"DFCG_DENSE_OP": "0", "DFCG_SPMM_SLAB": "1"},
    {"DFCG_DENSE_OP": "0", "DFCG_SPMM_CHUNK": "1"},
    {"DFCG_DENSE_OP": "0", "DFCG_SDDMM_TILE": "0"},
    {"DFCG_DENSE_OP": "0", "DFCG_SDDMM_SLAB": "0", "DFCG_SDDMM_TW": "1"},
    {"DFCG_DENSE_OP": "0", "DFCG_SDDMM_SLAB": "0", "DFCG_SDDMM_TW": "4"},
    {"DFCG_DENSE_OP": "0", "DFCG_SDDMM_SLAB": "1", "DFCG_SPMM_SLAB": "1"},
    {"DFCG_JACOBI_GRAPH": "1", "DFCG_JACOBI_CLUSTER": "1"},
    {"DFCG_JACOBI_PERSIST": "0"},
    {"DFCG_JACOBI_PERSIST": "1", "DFCG_JACOBI_CLUSTER": "1"},
    {"DFCG_JACOBI_PERSIST": "1", "DFCG_JACOBI_CLUSTER": "4"},
    {"DFCG_JACOBI_PERSIST": "1", "DFCG_JACOBI_NB": "16"},
    {"DFCG_JACOBI_PERSIST": "1", "DFCG_JACOBI_P2P": "1"},
    {"DFCG_JACOBI_PERSIST": "1", "DFCG_JACOBI_P2P": "1", "DFCG_JACOBI_CLUSTER": "2"},
    {"DFCG_DENSE_OP": "2", "DFCG_CHOLQR_SINGLE": "0"},
    {"DFCG_DENSE_OP": "2", "DFCG_CHOLQR_SINGLE": "1", "DFCG_CHOLQR_SINGLE_PIVOT": "1e-12"},
    {"DFCG_DENSE_OP": "2", "DFCG_CHOLQR_SINGLE": "1", "DFCG_CHOLQR_SINGLE_PIVOT": "0.5"},
    {"DFCG_CHOL_FUSED_MAXN": "100"},
    {"DFCG_DENSE_OP": "2", "DFCG_CHOLQR_WARM": "0"},
    {"DFCG_DENSE_OP": "2", "DFCG_CHOLQR_WARM_PIVOT": "0.999999"},
    {"DFCG_DENSE_OP": "0", "DFCG_SPMM16": "0"},
    {"DFCG_DENSE_OP": "0", "DFCG_SPMM16": "1", "DFCG_SPMM_CHUNK": "1"},
], ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()))
def test_variant_parity(env):
    r = subprocess.run([sys.executable, os.path.join(HERE, "_variant_case.py")], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
