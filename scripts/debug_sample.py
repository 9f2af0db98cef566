import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import make_cfg1, load_golden
from oracle import sampler as osamp
from paper_2601_04707_b200.graph import DeviceGraph
from paper_2601_04707_b200.cache import DeviceCache
from paper_2601_04707_b200.samplers import node_wise_block, PhiloxStream
gs = load_golden("sampling.npz")
hg = make_cfg1()
dg = DeviceGraph.from_csr(hg)
print("arcs", dg.num_arcs, dg.self_loops)
ro = dg.row_off.cpu().numpy(); col = dg.col.cpu().numpy()
print("strip ok", np.array_equal(ro, hg.row_offsets), np.array_equal(col, hg.col_indices))
mask = gs["cfg1/mask"]
c = DeviceCache(dg, mask)
ha = c.hot_arc[:c.num_hot_arcs].cpu().numpy(); ho = c.hot_off.cpu().numpy()
ref_hot = np.flatnonzero(mask[hg.col_indices])
print("hot arcs", c.num_hot_arcs, ref_hot.size, np.array_equal(ha, ref_hot))
ref_off = np.searchsorted(ref_hot, hg.row_offsets)
print("hot off", np.array_equal(ho, ref_off))
bits = c.bits.cpu().numpy().view(np.uint32)
unpack = ((bits[np.arange(10000)>>5] >> (np.arange(10000)&31)) & 1).astype(bool)
print("bits", np.array_equal(unpack, mask))
tg = gs["cfg1_b0/targets"]
for fan, m, cc in ((10, None, None), (10, mask, c)):
    blk = node_wise_block(dg, tg, fan, PhiloxStream(0,0,0,0), cached_mask=cc)
    ref = osamp.node_wise_block(hg.row_offsets, hg.col_indices, tg, fan, seed=0, epoch=0, batch_id=0, hop=0, cached_mask=m)
    r = blk.to_reference()
    print("fan", fan, "cache", m is not None, {k: np.array_equal(r[k], getattr(ref, k)) for k in ("rows","cols","src_ids")})
    # per-row compare
    rp = blk.row_ptr.cpu().numpy()
    rrows = ref.rows
    for i in range(len(tg)):
        a = r["src_ids"][r["cols"][rp[i]:rp[i+1]]]
        sel = np.flatnonzero(rrows == i)
        b = ref.src_ids[ref.cols[sel]]
        if not np.array_equal(a, b):
            v = tg[i]; nb = hg.col_indices[hg.row_offsets[v]:hg.row_offsets[v+1]]
            print("row", i, "v", v, "deg", nb.size, "hot", mask[nb].sum() if m is not None else None, "gpu", a, "ref", b)
            break
