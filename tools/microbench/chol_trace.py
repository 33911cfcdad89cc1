"""Critical-path breakdown of the tile Cholesky from an mb_chol_tiles trace (no U tasks, nt < 80).

Trace line: ticket t_start t_updates_done t_diag_staged t_compute_end t_published smid (ns).
For each diagonal task D_j prints: hop = t_diag_staged(D_j) - t_published(D_{j-1}) (the wait for
L_{j-1,j-1} and its L2 round trip), compute = t_compute_end - t_diag_staged (TRSM of (j, j-1),
rank-32 update, POTRF), publish = t_published - t_compute_end."""
import sys


def task_of(t, nt):
    c = start = 0
    while True:
        cnt = 1 + max(0, nt - c - 2)
        if t < start + cnt:
            break
        start += cnt
        c += 1
    return (0, c, c) if t == start else (1, c + 1 + (t - start), c)


def main(path, N):
    nt = (N + 31) // 32
    rows = [list(map(int, l.split())) for l in open(path)]
    base = min(r[1] for r in rows if r[1] > 0)
    for r in rows:  # times relative to the first task's start (entries past the last ticket stay 0)
        if r[1] > 0:
            r[1:6] = [v - base for v in r[1:6]]
    diag = {}
    for r in rows:
        typ, i, j = task_of(r[0], nt)
        if typ == 0:
            diag[j] = r
    hop = comp = pub = 0.0
    print("  j   start  upd_done  staged  comp_end  published   hop  compute  publish (us)")
    for j in range(nt):
        r = diag[j]
        h = (r[3] - diag[j - 1][5]) / 1e3 if j > 0 else 0.0
        c = (r[4] - r[3]) / 1e3
        p = (r[5] - r[4]) / 1e3
        hop += h
        comp += c
        pub += p
        if j < 4 or j % 8 == 0 or j > nt - 3:
            print(f"{j:3d} {r[1]/1e3:7.1f} {r[2]/1e3:8.1f} {r[3]/1e3:7.1f} {r[4]/1e3:8.1f} {r[5]/1e3:9.1f} {h:6.2f} {c:7.2f} {p:7.2f}")
    print(f"totals over {nt} steps: hop {hop:.1f} us, compute {comp:.1f} us, publish {pub:.1f} us; "
          f"end {diag[nt-1][5]/1e3:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2002)
