set -u
O=gpurun_out/r13
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 240 $R --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 --config bert_large --steps 5 --trace-dir $O/trace > $O/bert_n4_trace.json 2> $O/bert_n4_trace.err; echo t=$?
timeout 240 $R --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 --config bert_large --no-emulate > $O/bert_n4_noemu.json 2> $O/bert_n4_noemu.err; echo ne=$?
nvidia-smi topo -m > $O/topo.txt 2>&1
python - > $O/pcie_bw.txt 2>&1 <<'PY'
import torch, time
for dev in range(4):
    torch.cuda.set_device(dev)
    h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        f(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): f()
        b.record(); torch.cuda.synchronize()
        print(dev, name, round(10 * 256 * 2**20 / (a.elapsed_time(b) * 1e-3) / 1e9, 1), "GB/s")
PY
cat $O/pcie_bw.txt
