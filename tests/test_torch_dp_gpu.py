"""Real-backward producer: PyTorch autograd pushes gradients
into the KvStore from post-accumulate-grad hooks, step() pulls with the fused
SGD / momentum update, and the framework stream waits for the engine.

Checks, per step: the weights the model trains with are exactly the oracle
update (oracle/oracle.c or_sgd_update_f32 -- model.cpp:17-27 + momentum) of
the previous weights with the gradients autograd produced, and those
gradients are the ones a plain torch model computes from the same weights
(so the next forward really saw the updated weights)."""
import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_1802_06949_b200 import Engine, Transport  # noqa: E402
from paper_1802_06949_b200.torch_dp import TorchKvStoreDP  # noqa: E402


def _mlp(seed):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Linear(64, 256), torch.nn.ReLU(), torch.nn.Linear(256, 256),
                               torch.nn.ReLU(), torch.nn.Linear(256, 10)).cuda()


def _flat(ts):
    return np.concatenate([t.detach().float().cpu().numpy().ravel() for t in ts])


@pytest.mark.parametrize("bucket_mb", [0.0, 0.1, 25.0])
@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_torch_producer_single_gpu(gpu, bucket_mb, momentum):
    model = _mlp(0)
    ref = _mlp(0)
    eng = Engine(2, 0, None, 0)
    tr = Transport.local(1, 5000)
    lr, rescale = 0.05, 0.5
    dp = TorchKvStoreDP(model, eng, tr, 0, 1, lr=lr, momentum=momentum, rescale=rescale, bucket_mb=bucket_mb)
    if bucket_mb == 0.0:
        assert len(dp.groups) == len(dp.params)  # 1:1 comm_buf per key (kvstore.cpp:84)
    mom = np.zeros(sum(p.numel() for p in dp.params), np.float32)
    w = _flat(dp.params)
    gen = torch.Generator(device="cuda").manual_seed(1)
    for step in range(4):
        x = torch.randn(32, 64, device="cuda", generator=gen)
        y = torch.randint(0, 10, (32,), device="cuda", generator=gen)
        dp.zero_grad()
        loss = torch.nn.functional.cross_entropy(model(x), y)
        loss.backward()
        dp.step()
        torch.cuda.synchronize()
        g = _flat([p.grad for p in dp.params])
        # the gradient autograd produced is the one of the weights we hold
        with torch.no_grad():
            for pr, wv in zip(ref.parameters(), np.split(w, np.cumsum([p.numel() for p in dp.params])[:-1])):
                pr.copy_(torch.from_numpy(wv).view_as(pr))
        ref.zero_grad()
        torch.nn.functional.cross_entropy(ref(x), y).backward()
        np.testing.assert_allclose(g, _flat([p.grad for p in ref.parameters()]), rtol=1e-5, atol=1e-6)
        # and the weights are the oracle update of (w, g), bit for bit
        w, mom = O.sgd_update(w, g, lr, rescale, momentum, mom if momentum else None, kind="f32")
        if mom is None:
            mom = np.zeros_like(w)
        np.testing.assert_array_equal(_flat(dp.params), w, err_msg=f"step {step}")
    dp.close()
    eng.close()
    tr.close()


def test_torch_producer_requires_every_gradient(gpu):
    model = _mlp(0)
    eng = Engine(2, 0, None, 0)
    tr = Transport.local(1, 5000)
    dp = TorchKvStoreDP(model, eng, tr, 0, 1, bucket_mb=0.0)
    x = torch.randn(4, 64, device="cuda")
    dp.zero_grad()
    model[0](x).sum().backward()  # only the first layer gets gradients
    with pytest.raises(Exception, match="gradient buckets were pushed"):
        dp.step()
    dp.close()
    eng.close()
    tr.close()


@pytest.mark.parametrize("momentum", [0.0, 0.9])
def test_torch_producer_bucket_views(gpu, momentum):
    """bucket_views=True: autograd accumulates straight into the comm buckets
    (no pack copy); the weights are still the oracle update bit for bit."""
    model = _mlp(3)
    eng = Engine(2, 0, None, 0)
    tr = Transport.local(1, 5000)
    lr, rescale = 0.05, 0.5
    dp = TorchKvStoreDP(model, eng, tr, 0, 1, lr=lr, momentum=momentum, rescale=rescale, bucket_mb=0.1,
                        bucket_views=True)
    mom = np.zeros(sum(p.numel() for p in dp.params), np.float32)
    w = _flat(dp.params)
    gen = torch.Generator(device="cuda").manual_seed(5)
    for step in range(3):
        x = torch.randn(32, 64, device="cuda", generator=gen)
        y = torch.randint(0, 10, (32,), device="cuda", generator=gen)
        dp.zero_grad()
        torch.nn.functional.cross_entropy(model(x), y).backward()
        dp.step()
        torch.cuda.synchronize()
        g = _flat([p.grad for p in dp.params])  # 1 rank: the in-place "sum" is the gradient itself
        w, mom = O.sgd_update(w, g, lr, rescale, momentum, mom if momentum else None, kind="f32")
        if mom is None:
            mom = np.zeros_like(w)
        np.testing.assert_array_equal(_flat(dp.params), w, err_msg=f"step {step}")
    dp.close()
    eng.close()
    tr.close()
