"""B200-native SuperKMeans (arXiv 2603.20009): placeholder, API filled in below."""
