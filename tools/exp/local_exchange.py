"""Debug: LOCAL group halo exchange, 2 ranks on device 0."""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import torch
import paper_2310_01882_b200 as st

mode = sys.argv[1] if len(sys.argv) > 1 else "exchange"
comms = st.Comm.local_group(2)
streams = [torch.cuda.Stream() for _ in range(2)]
fs = [torch.full((6, 8), float(r + 1), dtype=torch.float64, device="cuda") for r in range(2)]
for r in range(2):
    comms[r].bind([fs[r]], 4)
torch.cuda.synchronize()
print("bound", flush=True)
for r in range(2):
    with torch.cuda.stream(streams[r]):
        st.st_halo_exchange(comms[r], [fs[r]], 4, 8, 1)
print("issued", flush=True)
t0 = time.time()
while time.time() - t0 < 10:
    q = [s.query() for s in streams]
    if all(q):
        break
    time.sleep(0.5)
print("streams done:", [s.query() for s in streams], flush=True)
if all(s.query() for s in streams):
    print(fs[0][:, 0].tolist(), fs[1][:, 0].tolist())
