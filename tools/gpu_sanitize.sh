# compute-sanitizer (memcheck / racecheck / synccheck) on small shapes of every kernel family
O=gpurun_out/sanitize
mkdir -p $O
cat > $O/small.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_1205_2926_b200 as ntt
P62, P30 = 29 * 2**57 + 1, 998244353
def run(p, bits, ell, batch, alg=3):
    L = 1 << ell
    plan = ntt.Plan(p, pow(3, (p - 1) // L, p), ell, bits, butterfly=alg)
    x = torch.empty(batch * L, dtype=torch.uint64 if bits == 64 else torch.uint32, device="cuda")
    ntt.synth_uniform(x, 1, ell, bound=p)
    plan.forward(x); plan.inverse(x) if alg == 3 else None
which = sys.argv[1] if len(sys.argv) > 1 else "all"
for p, bits, ell, batch in ((P62, 64, 12, 8), (P30, 32, 10, 4), (P62, 64, 15, 2), (P30, 32, 16, 2), (P62, 64, 18, 1), (P30, 32, 18, 1)):
    run(p, bits, ell, batch)
run(P62, 64, 18, 1, alg=5)
L = 1 << 16
plan = ntt.Plan(P30, pow(3, (P30 - 1) // L, P30), 16, 32)
a = torch.zeros(2 * L, dtype=torch.uint32, device="cuda"); b = torch.zeros_like(a)
ntt.synth_uniform(a, 1, 1, bits=20); ntt.synth_uniform(b, 1, 2, bits=20)
plan.cyclic_convolve(a, b)
torch.cuda.synchronize()
print("ok")
PY
which compute-sanitizer; compute-sanitizer --version | head -2
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python $O/small.py > $O/$tool.log 2>&1
  echo "$tool rc=$? $(tail -2 $O/$tool.log | tr '\n' ' ')"
done
