#!/bin/bash
# Tq=2 (NQ=128) attention time per source variant
C=paper_2510_12747_b200/csrc
mkdir -p /tmp/ab_orig && cp $C/*.cu $C/*.cuh /tmp/ab_orig/
for v in "$@"; do
  cp /tmp/ab_orig/* $C/ && cp $v/* $C/
  python -c "import paper_2510_12747_b200.build as b; b.build(force=True)" > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  python -c "
import sys; sys.path.insert(0,'tools'); import configs, paper_2510_12747_b200 as fv, torch
torch.cuda.set_device(0)
r=configs.run_point(rows=48, cols=88, heads=12, d=128, window=4, topk=36, mask=fv.Mask.all_allowed(), nq=2)
r2=configs.run_point(rows=48, cols=88, heads=12, d=128, window=4, topk=27, mask=fv.Mask.all_allowed(), nq=1)
print('$v tq2 attn_us %.1f  tq1 attn_us %.1f' % (r['attn_us'], r2['attn_us']))
" 2>&1 | tail -1
done
cp /tmp/ab_orig/* $C/
