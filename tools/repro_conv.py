import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, torch
import paper_1904_05347_b200 as tk, pyoracle as O
N,H,W,C,K,R,st,same = [int(v) for v in sys.argv[1].split(',')]
prec = sys.argv[2]
s = tk.ConvShape(N,H,W,C,K,R,R,st,bool(same)); conv = O.Conv(N,H,W,C,K,R,R,st,bool(same))
x = O.fill_random(int(np.prod(conv.in_shape)), 5).reshape(conv.in_shape)
f = O.fill_random(int(np.prod(conv.filt_shape)), 6).reshape(conv.filt_shape)
want = O.conv2d_naive(conv, x, f)
errs=[]
for i in range(6):
    dy = torch.full(s.out_shape, float('nan'), device='cuda')
    tk.conv2d_dev(torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda(), dy, s, tk.parse_conv_params('im2col'), precision=prec)
    torch.cuda.synchronize()
    g = dy.cpu().numpy()
    errs.append(O.max_scaled_error(g, want))
    if errs[-1] > 1e-2:
        bad = np.argwhere(np.abs(g - want) > 1e-2 * np.abs(want).max())
        print('bad count', len(bad), 'first', bad[:5].tolist(), 'of shape', g.shape)
print(sys.argv[1], prec, tk.conv2d_plan_info(s, tk.parse_conv_params('im2col'), prec)['kernel'], ['%.1e' % e for e in errs])
