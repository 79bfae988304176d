import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent.parent))
import torch
import paper_2310_01882_b200 as st
import stencil_inputs as si
m = 512
a = torch.from_numpy(si.jacobi3d_grid(m, m, m)).cuda()
b = torch.empty_like(a)
st.st_jacobi3d_run(a, b, 4, tblock=2)
torch.cuda.synchronize()
print("done")
