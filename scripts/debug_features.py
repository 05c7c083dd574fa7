import ctypes, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
from golden_cases import load_case
from paper_2409_02912_b200 import _lib
from paper_2409_02912_b200.nrx import noise_features, stack_pilots
c = load_case("c1_small")
n = c.y.shape[0]
geo = _lib.buffer_geometry(c.config, c.cfg, "fp32")
lib = _lib.load()
for yx, px in ((0,0),(1,0),(0,1),(1,1)):
    y = torch.from_numpy(c.y).to(torch.complex128 if yx else torch.complex64).cuda()
    p = torch.from_numpy(stack_pilots(c.books, n, c.cfg)).to(torch.complex128 if px else torch.complex64).cuda()
    nf = torch.from_numpy(noise_features(c.n0, n)).cuda()
    U = c.cfg.num_ues
    out = torch.zeros(n * U, geo["Cf"] // 4, geo["rows_slab"], 4, device="cuda")
    code = lib.nrx_ls_features(ctypes.byref(_lib.model_desc(c.config)), ctypes.byref(_lib.slot_desc(c.cfg)), n, 0,
                               y.data_ptr(), yx, p.data_ptr(), px, p.shape[0], nf.data_ptr(),
                               out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    f = out.cpu().numpy().transpose(0, 2, 1, 3).reshape(n * U, geo["rows_slab"], geo["Cf"])
    S, T = c.cfg.num_subcarriers, c.cfg.num_symbols
    f = f[:, :S * geo["Tp"]].reshape(n, U, S, geo["Tp"], geo["Cf"])[..., :T, :19]
    err = np.abs(f - c.features).max(axis=(0,1,2,3))
    print(yx, px, code, np.round(err, 7))
