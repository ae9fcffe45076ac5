"""CPU check of the distributed-storage address arithmetic shared by the Cholesky kernels
(`TileMap` / `RowSel` in paper_2405_14892_b200/csrc/common.cuh; __host__ __device__): the O(1)
closed forms of a rank's local tile index (1-D: owned tiles of the rows before i, a sum of a
periodic count; 2-D: the same over the rank's row blocks) and the row selection of the update
enumeration, against brute-force enumeration. Compiled for the host with nvcc (no GPU needed)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r'''
#include "common.cuh"
#include <cstdio>
int main() {
    using namespace mvn;
    long bad = 0, checked = 0;
    for (int P = 1; P <= 3; ++P) for (int Q = 1; Q <= 4; ++Q) for (int kp = 1; kp <= 8; kp += (kp < 3 ? 1 : 5))
    for (int pr = 0; pr < P; ++pr) for (int pc = 0; pc < Q; ++pc) for (int nt : {1, 5, 37}) {
        TileMap m = P == 1 ? TileMap::dist(nullptr, Q, pc, kp) : TileMap::dist2(nullptr, P, pr, Q, pc, kp);
        long cnt = 0;
        for (int i = 0; i < nt; ++i) for (int j = 0; j <= i; ++j)
            if ((j / kp) % Q == pc && (i / kp) % P == pr) { bad += m.index(i, j) != cnt; ++cnt; ++checked; }
        bad += m.index(nt, 0) != cnt;                       // the rank's tile count
        RowSel rs; rs.P = P; rs.pr = pr; rs.kp = kp; rs.lo = 3;
        for (int tj = 0; tj < nt; ++tj) {
            long c = 0;
            for (int i = tj > 3 ? tj : 3; i < nt; ++i)
                if ((i / kp) % P == pr) {
                    const long lo = tj > 3 ? tj : 3;
                    bad += rs.nth_raw(rs.raw(lo) + c) != i; ++c;
                }
            bad += upd_col_count(rs, nt, tj) != c;
        }
    }
    for (int k = 0; k < 9; ++k) for (int kp = 1; kp <= 8; ++kp) {   // the panel buffer layout
        TileMap m = TileMap::panel(nullptr, k, kp);
        long cnt = 0;
        for (int i = k; i < k + 30; ++i) for (int j = k; j <= (i < k + kp - 1 ? i : k + kp - 1); ++j) { bad += m.index(i, j) != cnt; ++cnt; }
    }
    printf("checked=%ld bad=%ld\n", checked, bad);
    return bad != 0;
}
'''


def test_tilemap_closed_forms(tmp_path):
    src = tmp_path / "tm.cu"
    src.write_text(SRC)
    exe = tmp_path / "tm"
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    subprocess.check_call([nvcc, "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-I",
                           os.path.join(ROOT, "paper_2405_14892_b200", "csrc"), "-o", str(exe), str(src)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bad=0" in r.stdout and "checked=0" not in r.stdout
