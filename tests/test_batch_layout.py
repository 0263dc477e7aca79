"""Host-side layout of batched scenes (no GPU): scenes per z column."""
from paper_1212_2845_b200.batch import y_stack_for, z_stack_for


def test_batch_z_stack_layout():
    assert z_stack_for(4096, 1) == 128          # 255 layers of cantilevers
    assert z_stack_for(64, 20) == 11            # 6 x blocks of 11 cubes (64 scenes)
    assert z_stack_for(32, 16) == 11            # 3 x blocks of 11 walkers
    assert z_stack_for(100, 40) == 1            # deep scenes: x only
    assert z_stack_for(1, 5) == 1
    for K in range(1, 300, 7):                  # every layout holds K scenes in <= 256 layers
        for nz in (1, 2, 5, 16, 20, 31):
            kz = z_stack_for(K, nz)
            assert 1 <= kz <= K and kz * (nz + 1) - 1 <= 256


def test_batch_y_stack_layout():
    assert y_stack_for(4096, 1, 1) == 128       # cantilevers: 255 rows of scenes
    assert y_stack_for(64, 20, 20) == 1         # a 20 x 20 plane already fills warps
    assert y_stack_for(5, 3, 4) == 5
    for K in range(1, 300, 7):
        for ny, nz in ((1, 1), (2, 3), (5, 5), (1, 31)):
            ky = y_stack_for(K, ny, nz)
            assert 1 <= ky <= K and ky * (ny + 1) - 1 <= 256
