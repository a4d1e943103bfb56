# Fast-path throughput vs problem size on one B200 (C4 and C3 families, ply count varied):
# how quickly k_combine reaches its HBM plateau.
for m in 4 8 16 32 64 128 192 256; do python tools/run_steps.py --config C4 --plies $m --steps 20; done
for m in 8 16 32 64 128; do python tools/run_steps.py --config C3 --plies $m --steps 20; done
