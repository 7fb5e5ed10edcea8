import sys, dataclasses, numpy as np, torch
sys.path.insert(0, '.')
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200 import _device
from tests.conftest import read_tle_pairs, GOLDEN
from paper_2603_27830_b200.tle import parse_catalog_columns
pairs = read_tle_pairs(GOLDEN / "leo_corpus.tle")[1]
corpus = parse_catalog_columns([a for a,_ in pairs],[b for _,b in pairs])
rng = np.random.default_rng(1)
n, m = int(rng.integers(1, 40)), int(rng.integers(1, 300))
cols = corpus[:, rng.integers(0, corpus.shape[1], n)]
times = np.sort(rng.uniform(-1440.0, 20160.0, m))
sats = pkg.init_batch(cols, precision=64)
res = pkg.propagate_batch(sats, times)
init = sats.init
col_init = dataclasses.replace(init, **{f.name: np.asarray(getattr(init, f.name))[:, None] for f in dataclasses.fields(init) if f.name not in ("grav", "dtype")})
st = pkg.sgp4_propagate(col_init, times)
a = np.moveaxis(st.r, -1, 0); b = res.planes[:3]
bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
idx = np.argwhere(bad.any(0))
print('n,m', n, m, 'bad cells', len(idx))
for i, j in idx[:10]:
    print(i, j, times[j], res.error[i, j], st.error_code[i, j], a[:, i, j], b[:, i, j])
# compare records: repacked vs original
dev2 = col_init._sgp4b_dev
r1 = sats.device_satrec.record.cpu().numpy(); r2 = dev2.record.cpu().numpy()
print('records equal', np.array_equal(r1.view(np.int64), r2.view(np.int64)))
d = np.argwhere(r1.view(np.int64) != r2.view(np.int64)); print(d[:10])
for k in d[:5]: print(k, r1[tuple(k)], r2[tuple(k)])
# pairs with original record
idx_d = torch.from_numpy(np.repeat(np.arange(n), m)).cuda(); t_d = torch.from_numpy(np.tile(times, n)).cuda()
rv = torch.empty((6, n*m), dtype=torch.float64, device='cuda'); c = torch.empty(n*m, dtype=torch.int32, device='cuda')
_device.propagate_pairs(sats.device_satrec, idx_d, t_d, rv, c)
rv = rv.cpu().numpy().reshape(6, n, m)
bad2 = ~((rv[:3] == b) | (np.isnan(rv[:3]) & np.isnan(b)))
print('pairs(orig record) vs grid bad', bad2.any(0).sum())
