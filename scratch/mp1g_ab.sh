python scratch/levels.py --tag group 2>&1 | tail -1
FT_MP1_CTA=1 python scratch/levels.py --tag cta 2>&1 | tail -1
