"""fp32 PyTorch restatement of the ResNet-50 chain (paper_2210_09603_b200/chain.py)
for the floating-point parity tests: the chain's own bf16 weights and input,
activations rounded to bf16 where the chain stores them."""


def stage_ref(chain, st, acts):
    """One stage from the activations in `acts` (name -> fp32 tensor)."""
    import torch
    F = torch.nn.functional
    r = lambda t: t.to(torch.bfloat16).float()  # noqa: E731
    x = acts[st.src]
    if st.kind == "conv":
        w, scale, shift = chain.params[st.dst]
        L = st.conv
        y = F.conv2d(x, w.float(), stride=L.s, padding=L.p)
        y = y * scale.view(1, -1, 1, 1) + shift.view(1, -1, 1, 1)
        if st.res:
            y = y + acts[st.res]
        if st.relu or st.res:
            y = torch.relu(y)
        return r(y)
    if st.kind == "maxpool":
        return F.max_pool2d(x, 3, 2, 1)
    if st.kind == "avgpool":
        return r(x.mean(dim=(2, 3)))
    wt, bias = chain.params[st.dst]
    return x @ wt.float() + bias


def chain_ref(chain):
    """The whole forward from the chain's input: name -> fp32 activation."""
    acts = {"input": chain.acts["input"].float()}
    for st in chain.stages:
        acts[st.dst] = stage_ref(chain, st, acts)
    return acts
