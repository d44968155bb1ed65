"""A training loop with lazy asynchronous checkpoints on one B200.

    python examples/train_loop.py [--steps 20] [--every 5] [--root /tmp/lzk_example]

What a trainer does with the engine (the reference's API: register shard
tensors, capture, lazy fence, persist, commit, restore):

  * the model parameters and Adam moments are registered ZERO-COPY
    (DeviceRegion.wrap on the live CUDA tensors);
  * capture() at the start of a checkpointed iteration returns in ~ms; the
    D2H snapshot runs on the copy engines behind forward/backward;
  * update_barrier_on_stream() makes the compute stream wait for the snapshot
    right before optimizer.step() mutates the tensors (no host blocking);
  * the flush persists the files in the background; commit() validates them
    on the GPU and records them in the manifest;
  * restore_into() brings a committed step back into the live tensors.

Checkpoints more frequent than the storage can absorb fill the pinned pool and
capture() then waits for the flush (the reference's backpressure). The pool
below holds six snapshots; with a 3 GB/s disk and a 0.4 GB state, one
checkpoint every ~10 ms still saturates it after a few (printed per step).
"""
import argparse
import os
import shutil
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10707_b200 as lz  # noqa: E402


def build_tree(model, opt):
    """Two top-level children = the two shard files of a 1-rank plan:
    a_params/* (layers file) and b_optim/* (optimizer file), as the
    reference's GPT example lays them out."""
    tree = lz.StateTree()
    for name, p in model.named_parameters():
        tree.set_region(f"a_params/{name}", lz.DeviceRegion.wrap(p.data))
    for name, p in model.named_parameters():
        st = opt.state[p]
        for k in ("exp_avg", "exp_avg_sq"):
            tree.set_region(f"b_optim/{name}/{k}", lz.DeviceRegion.wrap(st[k]))
    return tree


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--every", type=int, default=5)
    ap.add_argument("--root", default="/tmp/lzk_example")
    args = ap.parse_args()
    shutil.rmtree(args.root, ignore_errors=True)
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(4096, 4096), torch.nn.GELU(), torch.nn.Linear(4096, 4096)).cuda()
    opt = torch.optim.Adam(model.parameters(), lr=1e-3)
    x = torch.randn(256, 4096, device="cuda")
    loss = model(x).square().mean()  # one step so Adam's state exists
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=False)

    tree = build_tree(model, opt)
    params = sum(p.numel() for p in model.parameters())
    # plan: 4 B/param model file + 8 B/param (two Adam moments) optimizer file
    mspec = lz.ModelSpec(param_count=params, layer_count=1, bytes_per_param_model=4, bytes_per_param_optimizer=8)
    topo = lz.ParallelTopology(1, 1, 1, 1, 1)
    eng = lz.Engine(lz.EngineConfig(checkpoint_root=args.root, host_buffer_bytes=6 * tree.total_leaf_bytes() + (64 << 20)),
                    topo, lz.RankCoord())
    regions = [tree.region_at(l.path) for l in tree.flatten() if l.is_region]
    manifest = lz.ManifestStore(os.path.join(args.root, "manifest.json"))
    comp = torch.cuda.current_stream()
    tickets, losses = [], []
    t_start = time.perf_counter()
    for step in range(1, args.steps + 1):
        # no host synchronisation anywhere in the loop: capture() is ordered on
        # the device after the work already queued on `comp` (the previous
        # optimizer step), and the fence below orders the next one after the D2H
        ticket = (eng.capture(lz.plan_checkpoint(topo, mspec, step), tree, step, producer_stream=comp)
                  if step % args.every == 0 else None)
        loss = model(x).square().mean()          # forward + backward overlap the D2H
        loss.backward()
        if ticket is not None:
            eng.update_barrier_on_stream(ticket, comp.cuda_stream)  # lazy fence, device-side
        opt.step()                               # mutates the snapshotted tensors after the fence
        for r in regions:
            r.bump_version()                     # declare the in-place device mutation
        opt.zero_grad(set_to_none=False)
        if ticket is not None:
            tickets.append(ticket)
        losses.append((step, loss.detach(), ticket is not None))
    torch.cuda.synchronize()
    print(f"{args.steps} steps in {1e3 * (time.perf_counter() - t_start):.1f} ms (no host sync inside the loop)")
    for step, loss, ck in losses:
        print(f"step {step:3d} loss {loss.item():.5f}" + ("  [checkpoint]" if ck else ""))
    for t in tickets:
        ok, why = eng.commit(mspec, t, manifest)
        print(f"commit step {t.step()}: {'ok' if ok else why}")
    last = manifest.latest_committed()
    # restore the last committed step into the live tensors, then check it
    with torch.no_grad():
        for p in model.parameters():
            p.zero_()
    eng.restore_into(manifest, last, tree)
    torch.cuda.synchronize()
    back = eng.restore(manifest, last)
    exact = all(torch.equal(p.detach().view(torch.uint8).flatten().cpu(),
                            torch.frombuffer(bytearray(back.region_at(f"a_params/{n}").clone_bytes()),
                                             dtype=torch.uint8))
                for n, p in model.named_parameters())
    print(f"restored step {last}: in-place restore equals a fresh restore: {exact}")
    eng.close()
    shutil.rmtree(args.root, ignore_errors=True)
    return 0 if exact else 1


if __name__ == "__main__":
    sys.exit(main())
