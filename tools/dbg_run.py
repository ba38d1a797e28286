import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from inputs import synth
from tests.parity_util import run_parity
g = synth.generate(synth.CONFIGS["cfg1"])
print(run_parity(g, 2, 64, [10, 25], 256, 2500, 0.9, 4, 1.0, [1] * 12))
