import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2605_11381_b200 import fleet as fl, rounds, synthetic, _lib, device as dev
sizes=[100,5000]; k=300
soa = synthetic.fleet_soa(sum(sizes), seed=21)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, int(soa["issued_at"].min()))
fleet = fl.DeviceFleet.from_host(soa)
ref = rounds.DecisionRound(sum(sizes), k, sched)
ref.urgency(fleet); torch.cuda.synchronize()
keys = ref.keys.clone()
ku = keys.cpu().numpy().view(np.uint64)
order = np.lexsort((ku[:,1], ku[:,0]))
lib=_lib.load()
cands=[]
lo=0
for n in sizes:
    kk = keys[lo:lo+n].contiguous()
    kl = min(k, n)
    cand = fl.new_keys(k); cand.fill_(-1)
    ws = fl.Workspace(n)
    kthl = fl.new_keys(1)
    kth_ptr=None
    if kl < n:
        _lib.check(lib.kr_topk_select(kk.data_ptr(), n, kl, kthl.data_ptr(), None, ws.ptr(), ws.nbytes, dev.stream()), "sel")
        kth_ptr = kthl.data_ptr()
    _lib.check(lib.kr_admit(kk.data_ptr(), n, kl, kth_ptr, None, None, None, None, None, cand.data_ptr(), ws.ptr(), ws.nbytes, dev.stream()), "adm")
    torch.cuda.synchronize()
    cu = cand.cpu().numpy().view(np.uint64)
    sub = ku[lo:lo+n]; so = np.lexsort((sub[:,1], sub[:,0]))
    print('shard', lo, n, 'cand sorted == local topk:', np.array_equal(cu[:kl], sub[so[:kl]]), 'pad ok', (cu[kl:]==np.uint64(2**64-1)).all())
    cands.append(cand); lo+=n
g = torch.cat(cands)
m = g.shape[0]
wsm = fl.Workspace(m); kthg = fl.new_keys(1)
_lib.check(lib.kr_topk_select(g.data_ptr(), m, k, kthg.data_ptr(), None, wsm.ptr(), wsm.nbytes, dev.stream()), "selg")
torch.cuda.synchronize()
print('kth global == true kth:', np.array_equal(kthg.cpu().numpy().view(np.uint64)[0], ku[order[k-1]]))
print(kthg.cpu().numpy().view(np.uint64)[0], ku[order[k-1]])
gu = g.cpu().numpy().view(np.uint64); go = np.lexsort((gu[:,1], gu[:,0])); print('kth of gathered (numpy):', gu[go[k-1]])
