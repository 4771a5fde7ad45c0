"""Timeline of CTA 0 of the tcgen05 MLP kernel (DNNMG_MLP_TRACE=file): per A-ring
item (one K-chunk of one GEMM) the MMA issuer's wait start / a_full satisfied /
commit, and compute warp 0's arrive time; per GEMM the epilogue's acc_full time."""
import sys
import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64)
nk = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 8, 8, 8]
items = t[:6144].reshape(-1, 4)
acc = t[6144:6144 + 200]
n = int(np.argmax(items[:, 0] == 0)) if (items[:, 0] == 0).any() else len(items)
t0 = items[0, 0]
print("items", n)
g_per_tile = len(nk)
k = 0
j = 0
for tile in range(5):
    for g in range(g_per_tile):
        rows = items[k:k + nk[g]] - t0
        print(f"tile {tile} gemm {g}: epi acc_full@{acc[j] - t0 if acc[j] else -1}")
        for c, r in enumerate(rows):
            ae = t[8192 + k + c] - t0 if t.size > 8192 and t[8192 + k + c] else -1
            # hidden epilogues: tmem_ld issued / data ready / math done (warp 0)
            ls, lr, md = (t[b + k + c] - t0 if t[b + k + c] else -1 for b in (9216, 10240, 11264))
            ext = f" | ld@{ls:7d} ready+{lr - ls:4d} math+{md - lr:4d} slot+{ae - md:4d}" if ls >= 0 else ""
            print(f"   c{c}: mma_wait@{r[0]:7d} a_full@{r[1]:7d} (+{r[1]-r[0]:5d}) issued@{r[2]:7d} "
                  f"producer a_empty ok@{ae:7d} arrive@{r[3]:7d}{ext}")
        k += nk[g]
        j += 1
tot = items[n - 1, 2] - t0
print("per-tile cycles ~", (items[k, 0] - t0) / 3)
wait = (items[:n, 1] - items[:n, 0]).sum()
print(f"MMA waiting on a_full: {wait} of {tot} cycles ({100 * wait / tot:.1f}%)")
commit = t[6400:6400 + 200]
before = t[6656:6656 + 200]
print("per GEMM j: MMA commit(acc_full) | epi arrives at wait | epi wait returns")
for jj in range(12):
    print(f"  j{jj}: commit@{commit[jj] - t0:7d} epi_at_wait@{before[jj] - t0:7d} returns@{acc[jj] - t0:7d}")
tl = t[6912:6912 + 40].reshape(-1, 4)
for i in range(3):
    print(f"tile {i}: load_x start@{tl[i,0]-t0} end@{tl[i,1]-t0} head epi done@{tl[i,2]-t0} "
          f"stage ready (tile {i})@{tl[i,3]-t0 if tl[i,3] else -1}")
