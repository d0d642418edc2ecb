import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch, torch.nn.functional as Fn
from paper_2208_14228_b200 import resnet as rn
import test_gpu_resnet as T
job = rn.ResNetJob(gpus=1, ests=2, batch=4, seed=7)
P = T._d(job.params).clone().requires_grad_(True)
cap = {}
losses = job.step(capture=cap)
E, B = job.E, job.B
img = T._nchw(cap["img"], E * B, 32, 8)
labels = cap["labels"].long().cpu()
# restatement with hooks on the last block
saved = {}
eps = job.eps
N = E * B
def bn(z, cv, relu=True, res=None):
    g0, b0 = job.off[cv.name][1:]
    zz = z.view(E, B, cv.co, -1).transpose(1, 2).reshape(E, cv.co, -1)
    m = zz.mean(-1).repeat_interleave(B, 0).view(N, cv.co, 1, 1)
    v = zz.var(-1, unbiased=False).repeat_interleave(B, 0).view(N, cv.co, 1, 1)
    y = P[g0:g0 + cv.co].view(1, -1, 1, 1) * (z - m) / torch.sqrt(v + eps) + P[b0:b0 + cv.co].view(1, -1, 1, 1)
    if res is not None: y = y + res
    return T._bf(torch.relu(y) if relu else y)
def conv(x, cv):
    w0 = job.off[cv.name][0]
    w = P[w0:w0 + cv.co * cv.K].view(cv.co, cv.k, cv.k, cv.ci).permute(0, 3, 1, 2)
    return T._bf(Fn.conv2d(x, T._bf(w), stride=cv.s, padding=cv.p))
x = bn(conv(img, job.convs[0]), job.convs[0])
for a, b, d in job.blocks:
    h = bn(conv(x, a), a)
    res = x if d is None else bn(conv(x, d), d, relu=False)
    zb = conv(h, b); zb.retain_grad(); saved['zb'] = zb; saved['h'] = h
    x = bn(zb, b, res=res)
x.retain_grad()
pooled = x.mean((2, 3))
fw, fb = job.off_fc
logits = pooled @ P[fw:fw + 5120].view(10, 512).T + P[fb:fb + 10]
ce = Fn.cross_entropy(logits, labels, reduction="none").view(E, B).mean(1)
ce.sum().backward()
print('loss', losses, ce)
top = T._nchw(cap['top'], N, 4, 512)
print('top rel', float((top - x.detach()).norm() / x.detach().norm()))
dtop = T._nchw(cap['dtop'], N, 4, 512)
print('dtop rel', float((dtop - x.grad).norm() / x.grad.norm()))
lo, hi = job.off['l4.1.b'][0], job.off['l4.1.b'][1]
g = cap['grads'].double().cpu()
gsum = g[0] + g[1]
print('W l4.1.b rel', float((gsum[lo:hi] - P.grad[lo:hi]).norm() / P.grad[lo:hi].norm()))
g0_, b0_ = job.off['l4.1.b'][1:]
print('gamma rel', float((gsum[g0_:g0_+512] - P.grad[g0_:g0_+512]).norm() / P.grad[g0_:g0_+512].norm()))
print('beta rel', float((gsum[b0_:b0_+512] - P.grad[b0_:b0_+512]).norm() / P.grad[b0_:b0_+512].norm()))
for nm in ['l4.1.a', 'l4.0.b', 'l4.0.d', 'l3.1.b', 'stem']:
    lo, hi = job.off[nm][0], job.off[nm][1]
    print(nm, 'W rel', float((gsum[lo:hi] - P.grad[lo:hi]).norm() / P.grad[lo:hi].norm()))
# direct dW check from saved zb grad and h
zbg = saved['zb'].grad  # [N][512][4][4]
hcol = Fn.unfold(saved['h'].detach(), 3, padding=1)  # [N][512*9][16] ordering (c, kh, kw)
dW = torch.einsum('nop,nkp->ok', zbg.view(N, 512, 16), hcol).view(512, 512, 3, 3).permute(0, 2, 3, 1).reshape(-1)
print('dW from autograd zb.grad vs P.grad', float((dW - P.grad[job.off['l4.1.b'][0]:job.off['l4.1.b'][1]]).norm() / dW.norm()))
