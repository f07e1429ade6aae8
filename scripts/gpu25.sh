./tools/tile_micro
