"""Writes the closed-form E[<x_bar, x>] values in hand_values.json.

For x uniform on the unit sphere of R^d and the sign codebook {+-1/sqrt(d)}^d
(PAPER P:243), <x_bar, x> = sum_j |x_j| / sqrt(d), and E|x_j| =
Gamma(d/2) / (sqrt(pi) Gamma((d+1)/2)), so E[u] = sqrt(d) Gamma(d/2) /
(sqrt(pi) Gamma((d+1)/2)).  Pure mathematics: calls nothing but math.
"""
from math import exp, lgamma, pi, sqrt

if __name__ == "__main__":
    for d in (16, 32, 64, 128, 256, 512):
        print(d, sqrt(d) * exp(lgamma(d / 2) - lgamma((d + 1) / 2)) / sqrt(pi))
