bash tools/ab.sh FVSR_ATTN_EXP=19 FVSR_ATTN_EXP=1
FVSR_ATTN_EXP=19 FVSR_ATTN_INSTRUMENT=1 python -c "import paper_2510_12747_b200.build as b; b.build(force=True)" > /dev/null 2>&1
FVSR_ATTN_TRACE=1 python bench.py --steps 30 --warmup 10 --no-cpu --e2e-steps 1 > /dev/null 2> gpurun_out/trace_skel.txt
