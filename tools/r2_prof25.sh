mkdir -p gpurun_out
BS_K5_PAIR=1 timeout 300 python tools/k5_pair_check.py /tmp/pair.pt > gpurun_out/r2_pair25.txt 2>&1; echo "pair rc=$?"
BS_K5_PAIR=0 timeout 300 python tools/k5_pair_check.py /tmp/single.pt >> gpurun_out/r2_pair25.txt 2>&1; echo "single rc=$?"
python -c "
import torch
a=torch.load('/tmp/pair.pt'); b=torch.load('/tmp/single.pt')
for k in a: print(k, 'bit-identical' if torch.equal(a[k],b[k]) else 'DIFFERENT', (a[k].float()-b[k].float()).abs().max().item())
" >> gpurun_out/r2_pair25.txt 2>&1
cat gpurun_out/r2_pair25.txt
for p in 1 0; do BS_K5_PAIR=$p timeout 600 python tools/tc_probe.py sp24_16384 sp24_ctc_ih | sed "s/^/pair=$p /" >> gpurun_out/r2_tc25.txt 2>&1; done
BS_K5_RT=1 timeout 600 python tools/tc_probe.py sp24_16384 sp24_ctc_ih | sed "s/^/rt=1 /" >> gpurun_out/r2_tc25.txt 2>&1
cat gpurun_out/r2_tc25.txt
