"""Forward attention time at few heads per GPU for forced KV-split chunk sizes."""
import os, sys, json, subprocess
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_2411_15871_b200 import device as dh
    T, nq, nkv, d = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), 128
    qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
    o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    f = lambda: dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, d ** -0.5)  # noqa: E731
    for _ in range(3): f()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(20): f()
    e.record(); torch.cuda.synchronize()
    print(s.elapsed_time(e) / 20 * 1e3)
    sys.exit(0)
for T, nq, nkv in ((4096, 4, 1), (4096, 8, 2), (8192, 4, 1)):
    row = {}
    for ch in ("auto", "0", "4", "6", "8", "12", "16"):
        env = dict(os.environ)
        if ch != "auto":
            env["DH_ATTN_FWD_CHUNK"] = ch if ch != "0" else "9999"
        r = subprocess.run([sys.executable, __file__, "child", str(T), str(nq), str(nkv)], env=env,
                           capture_output=True, text=True)
        row[ch] = round(float(r.stdout.strip().splitlines()[-1]), 1) if r.returncode == 0 else r.stderr[-200:]
    print(json.dumps({"T": T, "nq": nq, "us": row}), flush=True)
