"""Plain PyTorch fp32 reference of the GPT-2 step the B200 executor runs (test infrastructure;
used only to check the CUDA path numerically). Parameter layout = BlockLayout in
paper_2503_01890_b200/csrc/runtime/gpt_model.h."""
import math

import torch
import torch.nn.functional as F


def block_slices(h):
    out, at = {}, 0
    for name, shape in (("w_qkv", (3 * h, h)), ("w_proj", (h, h)), ("w_fc", (4 * h, h)), ("w_fc2", (h, 4 * h)),
                        ("b_qkv", (3 * h,)), ("b_proj", (h,)), ("b_fc", (4 * h,)), ("b_fc2", (h,)),
                        ("ln1_g", (h,)), ("ln1_b", (h,)), ("ln2_g", (h,)), ("ln2_b", (h,))):
        n = math.prod(shape)
        out[name] = (at, shape)
        at += n
    assert at == 12 * h * h + 13 * h
    return out


def unflatten(flat, h):
    return {k: flat[a:a + math.prod(s)].view(*s) for k, (a, s) in block_slices(h).items()}


def flatten_grads(grads, h):
    out = torch.zeros(12 * h * h + 13 * h, dtype=torch.float32)
    for k, (a, s) in block_slices(h).items():
        out[a:a + math.prod(s)] = grads[k].reshape(-1)
    return out


def block_fwd(x, W, nh):
    B, s, h = x.shape
    hd = h // nh
    a = F.layer_norm(x, (h,), W["ln1_g"], W["ln1_b"], eps=1e-5)
    qkv = a @ W["w_qkv"].T + W["b_qkv"]
    q, k, v = qkv.split(h, dim=-1)
    q = q.view(B, s, nh, hd).transpose(1, 2)
    k = k.view(B, s, nh, hd).transpose(1, 2)
    v = v.view(B, s, nh, hd).transpose(1, 2)
    att = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    att = att.transpose(1, 2).reshape(B, s, h)
    x2 = x + att @ W["w_proj"].T + W["b_proj"]
    m = F.layer_norm(x2, (h,), W["ln2_g"], W["ln2_b"], eps=1e-5)
    m = F.gelu(m @ W["w_fc"].T + W["b_fc"], approximate="tanh")
    return x2 + m @ W["w_fc2"].T + W["b_fc2"]


def loss_and_grads(blocks, wte, wpe, lnf, tokens, targets, nh, V):
    """blocks: list of flat fp32 tensors; wte [Vp, h]; wpe [s, h]; lnf [2h]. Returns (loss, grads)."""
    h = wte.shape[1]
    params = [b.clone().requires_grad_(True) for b in blocks]
    wte_ = wte.clone().requires_grad_(True)
    wpe_ = wpe.clone().requires_grad_(True)
    lnf_ = lnf.clone().requires_grad_(True)
    B, s = tokens.shape
    x = wte_[tokens] + wpe_[torch.arange(s, device=tokens.device)]
    for p in params:
        x = block_fwd(x, unflatten(p, h), nh)
    x = F.layer_norm(x, (h,), lnf_[:h], lnf_[h:], eps=1e-5)
    logits = (x @ wte_.T)[..., :V]
    loss = F.cross_entropy(logits.reshape(-1, V), targets.reshape(-1))
    loss.backward()
    return loss.item(), [p.grad for p in params], wte_.grad, wpe_.grad, lnf_.grad
