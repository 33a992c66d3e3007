"""Profiling driver (ncu target): a few eager CIFAR-10-quick training steps
through the public API, so every kernel of the step appears in order.
Usage: python profiles/prof_step.py [steps] [cifar10_quick|alexnet|lenet|resnet20]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02272_b200 import polegrad  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
model = sys.argv[2] if len(sys.argv) > 2 else "cifar10_quick"
shape = {"cifar10_quick": (100, 3, 32, 32, 10), "alexnet": (256, 3, 227, 227, 1000), "lenet": (64, 1, 28, 28, 10),
         "resnet20": (128, 3, 32, 32, 10)}[model]
net = polegrad.Net(polegrad.load_model(model), seed=1, dtype="f32")
solver = polegrad.Solver(net, method="sgd", lr=0.001, momentum=0.9, weight_decay=0.004)
rng = np.random.default_rng(2)
x = rng.uniform(-1, 1, shape[:4]).astype(np.float32)
y = np.floor(rng.uniform(0, 1, shape[0]) * shape[4]).astype(np.float32)
for _ in range(steps):
    net.set_batch(x, y)
    net.forward()
    net.backward()
    solver.apply()
net.sync()
print("loss", net.loss())
