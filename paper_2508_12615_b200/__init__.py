"""WIPES wavelet differentiable rasterizer — B200-native (sm_100a) hot path."""
